#!/bin/bash
# backward_weight pair-step candidates (O1D_PPSTEPS 16 vs 4) + parity subset + per-angle
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dp_gpu.py -m gpu -q -x -n 3 -k "full_stage1 or assignments_spec or angle_sets_spec or stage1_like_ragged or repeated or step_api or flat_16bit or fused or dp or 1dpp or shear or bilinear" 2>&1 | tail -2
for e in 16 4 16 4; do
  O1D_PPSTEPS=$e timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu --no-e2e --no-extra > gpurun_out/pp.json 2>&1; echo "PPSTEPS=$e f32 $(python tools/bench_brief.py gpurun_out/pp.json | cut -c1-200)"
done
O1D_PPSTEPS=16 timeout 300 python bench.py --dtype bf16 --steps 300 --warmup 5 --no-cpu --no-e2e --no-extra > gpurun_out/pp.json 2>&1; echo "PPSTEPS=16 bf16 $(python tools/bench_brief.py gpurun_out/pp.json | cut -c1-200)"
bash tools/angles.sh
