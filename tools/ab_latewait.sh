#!/bin/bash
# late band-store wait A/B (O1D_LATEWAIT) + stencil parity subset
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -n 3 -k "full_stage1 or assignments_spec or angle_sets_spec or stage1_like_ragged or repeated or step_api or flat_16bit or fused or 1dpp or outputs_fully" 2>&1 | tail -2
for e in 1 0 1 0; do
  O1D_LATEWAIT=$e timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu --no-e2e --no-extra > gpurun_out/lw.json 2>&1; echo "LATEWAIT=$e f32 $(python tools/bench_brief.py gpurun_out/lw.json | cut -c1-200)"
done
for e in 1 0; do
  O1D_LATEWAIT=$e timeout 300 python bench.py --dtype bf16 --steps 300 --warmup 5 --no-cpu --no-e2e --no-extra > gpurun_out/lw.json 2>&1; echo "LATEWAIT=$e bf16 $(python tools/bench_brief.py gpurun_out/lw.json | cut -c1-200)"
done
