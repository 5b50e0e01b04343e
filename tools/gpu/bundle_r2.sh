#!/bin/bash
# Round-2 evidence bundle (one gpurun call): smoke, GPU suite, default bench line (cpu baseline, e2e,
# extras), K-sweep lines, per-angle runs, launch list, ncu --set full captures.  Outputs in gpurun_out/.
TAG=${1:-r2z}; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1; echo smoke rc $?
timeout 1800 python -m pytest tests -m gpu -q --timeout 1200 -n 3 > gpurun_out/gpu_tests_$TAG.txt 2>&1; echo tests rc $?; tail -2 gpurun_out/gpu_tests_$TAG.txt
timeout 1200 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc $?
python tools/bench_brief.py gpurun_out/bench_$TAG.json
for K in 7 15 23 31 39 47 55 63; do
  timeout 300 python bench.py --workload ks --K $K --steps 100 --warmup 5 --no-extra --no-e2e --no-cpu > gpurun_out/ks_${K}_$TAG.json 2>/dev/null
  echo "K=$K $(python tools/bench_brief.py gpurun_out/ks_${K}_$TAG.json 2>&1 | head -1)"
done > gpurun_out/ksweep_$TAG.txt
for a in 0 22.5 45 67.5 90 112.5 135 157.5; do
  timeout 300 python bench.py --steps 50 --warmup 3 --no-extra --no-e2e --no-cpu --angle $a 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('angle $a', round(d['value']), {k: round(v*1000,1) for k,v in d['per_pass_ms'].items()})"
done > gpurun_out/angles_$TAG.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extra > /dev/null 2>&1; echo launches rc $?
ncu --set full --clock-control none --import-source on -k regex:o1d_ -s 8 -c 4 -o gpurun_out/full_$TAG \
    python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-extra > /dev/null 2>&1; echo full rc $?
ncu --set full --clock-control none --import-source on -k regex:o1d_stencil -s 4 -c 1 -o gpurun_out/full_bf16_$TAG \
    python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-extra --dtype bf16 > /dev/null 2>&1; echo bf16 rc $?
ncu --set full --clock-control none --import-source on -k regex:o1d_small -s 3 -c 3 -o gpurun_out/small_$TAG \
    python bench.py --workload ks --K 31 --steps 2 --warmup 1 --no-e2e --no-cpu --no-extra > /dev/null 2>&1; echo small rc $?
cat gpurun_out/ksweep_$TAG.txt gpurun_out/angles_$TAG.txt
