python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "stride or generic or ragged or tiny" -n 3 2>&1 | tail -2
for args in "128 64 224 224 5 2 0 bf16" "128 64 112 112 5 1 90 bf16" "128 64 112 112 5 2 90 bf16"; do
  timeout 120 python tools/layer_bench.py $args 2>&1 | tail -1; done
timeout 600 python bench.py --model convnext_t_1d --steps 10 --warmup 3 2>&1 | tail -1 | cut -c1-300
