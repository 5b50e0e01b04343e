#!/bin/bash
# Round-2 profiling: launch list of the default bench, one ncu --set full capture per pass
# kernel (fp32 S1, plus the bf16 forward), per-angle times.  usage: gpurun -- bash tools/prof_r2.sh TAG
TAG=${1:-r2}; mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extra > /dev/null 2>&1; echo launches rc $?
# kernels in bench order per step: stencil(fwd) stencil(bwd_in) wgrad finalize; skip warm-up launches
ncu --set full --clock-control none --import-source on -k regex:o1d_ -s 8 -c 4 -o gpurun_out/full_$TAG \
    python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-extra > /dev/null 2>&1; echo full rc $?
ncu --set full --clock-control none --import-source on -k regex:o1d_stencil -s 4 -c 1 -o gpurun_out/full_bf16_$TAG \
    python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-extra --dtype bf16 > /dev/null 2>&1; echo bf16 rc $?
for a in 0 22.5 45 67.5 90 112.5 135 157.5; do
  timeout 300 python bench.py --steps 30 --warmup 3 --no-extra --no-e2e --no-cpu --angle $a 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('angle $a', round(d['value']), {k: round(v*1000,1) for k,v in d['per_pass_ms'].items()})"
done > gpurun_out/angles_$TAG.txt 2>&1
cat gpurun_out/angles_$TAG.txt
