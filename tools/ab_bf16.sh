#!/bin/bash
# bf16 change check (under gpurun): 16-bit parity subset, then bf16 and f32 bench lines
TAG=${1:-x}; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dp_gpu.py -m gpu -q -x -n 3 -k "full_stage1_config or stage1_like_ragged or assignments_spec or bilinear_full or outputs_fully or step_api or repeated or fused or tiny or dp" > gpurun_out/bf16_tests_$TAG.txt 2>&1; echo tests rc $?; tail -3 gpurun_out/bf16_tests_$TAG.txt
for a in "--dtype bf16" "--dtype f32"; do
  timeout 300 python bench.py $a --steps 200 --warmup 5 --no-cpu --no-e2e --no-extra > gpurun_out/ab_$TAG.json 2>gpurun_out/ab_$TAG.err
  echo "$a"; python tools/bench_brief.py gpurun_out/ab_$TAG.json || tail -5 gpurun_out/ab_$TAG.err
done
