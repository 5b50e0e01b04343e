#!/bin/bash
# o1d_step pass order A/B (O1D_STEP_ORDER: 0 forward first, 1 backward_weight first)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "step" 2>&1 | tail -1
O1D_STEP_ORDER=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "step" 2>&1 | tail -1
for r in 1 2 3; do for e in 1 0; do
  O1D_STEP_ORDER=$e timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu --no-e2e --no-extra > gpurun_out/ord.json 2>&1; echo "ORDER=$e f32 $(python tools/bench_brief.py gpurun_out/ord.json | cut -c1-130)"
done; done
for e in 1 0; do O1D_STEP_ORDER=$e timeout 300 python bench.py --dtype bf16 --steps 300 --warmup 5 --no-cpu --no-e2e --no-extra > gpurun_out/ord.json 2>&1; echo "ORDER=$e bf16 $(python tools/bench_brief.py gpurun_out/ord.json | cut -c1-130)"; done
