python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "small_planes or ksweep or tiny or ragged or fully" -n 3 2>&1 | tail -2
for args in "128 768 7 7 15 1 D8 bf16" "128 768 7 7 15 1 D8 f32"; do timeout 120 python tools/layer_bench.py $args 2>&1 | tail -1; done
timeout 600 python bench.py --model convnext_t_1d --steps 10 --warmup 3 2>&1 | tail -1 | cut -c1-200
