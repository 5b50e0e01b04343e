python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "small_planes or ksweep or tiny" -n 3 2>&1 | tail -2
for K in 7 31 63; do timeout 300 python bench.py --workload ks --K $K --steps 100 --warmup 5 --no-extra --no-e2e --no-cpu > /tmp/ks.json 2>/tmp/ks.err; echo "K=$K $(python tools/bench_brief.py /tmp/ks.json || tail -5 /tmp/ks.err)"; done
