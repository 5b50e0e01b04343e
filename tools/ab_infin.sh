#!/bin/bash
# in-kernel backward_weight finalize (O1D_INFIN, cooperative launch) A/B + the tests that touch backward_weight
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_dp_gpu.py -m gpu -q -x -n 3 -k "full_stage1 or assignments_spec or angle_sets_spec or stage1_like_ragged or repeated or step or fused or dp or 1dpp or concurrent or opcheck or autograd or convnext or flat or bilinear or shear or outputs_fully" 2>&1 | tail -2
for e in 1 0 1 0; do
  O1D_INFIN=$e timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu --no-e2e --no-extra > gpurun_out/inf.json 2>&1; echo "INFIN=$e f32 $(python tools/bench_brief.py gpurun_out/inf.json | cut -c1-230)"
done
for e in 1 0; do
  O1D_INFIN=$e timeout 300 python bench.py --dtype bf16 --steps 300 --warmup 5 --no-cpu --no-e2e --no-extra > gpurun_out/inf.json 2>&1; echo "INFIN=$e bf16 $(python tools/bench_brief.py gpurun_out/inf.json | cut -c1-230)"
done
