#!/bin/bash
# Round-2 evidence bundle (run under gpurun): default bench line, launch list, ncu full captures (fp32 passes,
# bf16 stencil + wgrad, small-plane K=31), per-angle runs, K-sweep, model line, GPU tests, smoke.
# usage: gpurun -- bash tools/bundle_r2.sh TAG      (outputs in gpurun_out/)
TAG=${1:-r2}; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1; echo smoke rc $?
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc $?
python tools/bench_brief.py gpurun_out/bench_$TAG.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extra > /dev/null 2>&1; echo launches rc $?
ncu --set full --clock-control none --import-source on -k regex:o1d_ -s 8 -c 4 -o gpurun_out/full_$TAG \
    python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-extra > /dev/null 2>&1; echo full rc $?
ncu --set full --clock-control none --import-source on -k regex:o1d_ -s 8 -c 3 -o gpurun_out/full_bf16_$TAG \
    python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-extra --dtype bf16 > /dev/null 2>&1; echo bf16 rc $?
ncu --set full --clock-control none --import-source on -k regex:o1d_small -s 6 -c 3 -o gpurun_out/full_ks31_$TAG \
    python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-extra --workload ks --K 31 > /dev/null 2>&1; echo ks rc $?
for f in full_$TAG full_bf16_$TAG full_ks31_$TAG; do python tools/ncu_summary.py gpurun_out/$f.ncu-rep > gpurun_out/${f}_summary.txt 2>&1; done
python tools/traffic_json.py gpurun_out/full_$TAG.ncu-rep gpurun_out/traffic_$TAG.json > /dev/null 2>&1
bash tools/angles.sh > gpurun_out/angles_$TAG.txt 2>&1
for K in 7 15 23 31 39 47 55 63; do
  timeout 300 python bench.py --workload ks --K $K --steps 50 --warmup 5 --no-cpu --no-e2e --no-extra > gpurun_out/ks.json 2>&1
  echo "K=$K $(python tools/bench_brief.py gpurun_out/ks.json)"
done > gpurun_out/ksweep_$TAG.txt 2>&1
timeout 900 python bench.py --model convnext_t_1d --steps 20 --warmup 5 > gpurun_out/model_$TAG.json 2>&1; echo model rc $?
timeout 1800 python -m pytest tests -m gpu -q --timeout 1200 -n 3 > gpurun_out/gpu_tests_$TAG.txt 2>&1; echo tests rc $?
tail -2 gpurun_out/gpu_tests_$TAG.txt; tail -1 gpurun_out/smoke_$TAG.txt | cut -c1-200
