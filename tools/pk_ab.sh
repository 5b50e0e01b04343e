#!/bin/bash
# A/B of the packed 16-bit rings (O1D_PK stencil, O1D_PKW backward_weight) at S1 bf16, plus bf16 parity tests
# usage (under gpurun): bash tools/pk_ab.sh TAG
TAG=${1:-x}; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for p in 0 1 2; do timeout 120 python tools/debug_spec.py 2 16 56 56 31 $p bf16 2>&1 | grep -v "^\s*$" | tail -1 | cut -c1-150; done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "full_stage1_config or stage1_like_ragged or assignments_spec or bilinear_full or outputs_fully or small_planes or step_api or repeated" > gpurun_out/pk_tests_$TAG.txt 2>&1; echo tests rc $?; tail -3 gpurun_out/pk_tests_$TAG.txt
for cfg in "O1D_PK=1 O1D_PKW=1" "O1D_PK=0 O1D_PKW=0" "O1D_PK=1 O1D_PKW=0"; do
  env $cfg timeout 300 python bench.py --dtype bf16 --steps 200 --warmup 5 --no-cpu --no-e2e --no-extra > gpurun_out/pk_$TAG.json 2>gpurun_out/pk_$TAG.err
  echo "$cfg"; python tools/bench_brief.py gpurun_out/pk_$TAG.json || tail -5 gpurun_out/pk_$TAG.err
done
