#!/bin/bash
# scheduler claim-ahead (O1D_PREF: single-item atomics in flight per producer; 0 = claim when a slot frees)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_dp_gpu.py -m gpu -q -x -n 3 -k "full_stage1 or assignments_spec or angle_sets_spec or stage1_like_ragged or repeated or step or fused or dp or 1dpp or concurrent or flat or bilinear_full or outputs_fully" 2>&1 | tail -2
for r in 1 2 3; do for e in 0 2; do
  O1D_PREF=$e timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu --no-e2e --no-extra > gpurun_out/pref.json 2>&1; echo "PREF=$e f32 $(python tools/bench_brief.py gpurun_out/pref.json | cut -c1-230)"
done; done
for e in 0 2; do
  O1D_PREF=$e timeout 300 python bench.py --dtype bf16 --steps 300 --warmup 5 --no-cpu --no-e2e --no-extra > gpurun_out/pref.json 2>&1; echo "PREF=$e bf16 $(python tools/bench_brief.py gpurun_out/pref.json | cut -c1-230)"
done
O1D_PREF=0 bash tools/angles.sh
