#!/bin/bash
# Round profiling bundle (run under gpurun): bench line, launch list, full ncu capture,
# per-angle uniformity, clocks.  Outputs land in gpurun_out/.
set -x
TAG=${1:-r1}
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extra > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:o1d_ -s 4 -c 4 -o gpurun_out/full_$TAG \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-extra > /dev/null 2>&1
./tools/angles.sh > gpurun_out/angles_$TAG.txt 2>&1
O1D_TRACE=1 TRACE_TABLES=1 TRACE_LAT=1 timeout 300 python tools/trace_pass.py > gpurun_out/trace_$TAG.txt 2>&1
python tools/rep_check.py 300 > gpurun_out/repcheck_$TAG.txt 2>&1
python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-extra --flags 1 > gpurun_out/bench_generic_$TAG.json 2>&1
