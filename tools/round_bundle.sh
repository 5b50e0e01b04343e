#!/bin/bash
# Round-end evidence bundle (run under gpurun): profile_round.sh + GPU tests + smoke
# usage: gpurun -- bash tools/round_bundle.sh <tag>
mkdir -p gpurun_out; TAG=${1:-r1l}
timeout 1500 bash tools/profile_round.sh $TAG > gpurun_out/profile_$TAG.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_$TAG.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$TAG.txt 2>&1
tail -2 gpurun_out/gpu_tests_$TAG.txt; cat gpurun_out/smoke_$TAG.txt | tail -2
