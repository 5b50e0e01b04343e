#!/bin/bash
# flat 16-bit planes: parity + the ConvNeXt stage-2 layer timing (spec vs forced generic)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "flat_16bit or full_stage1_config or assignments_spec" 2>&1 | tail -4
for f in 0 1; do timeout 300 python tools/layer_bench.py 128 192 28 28 31 1 D8 bf16 $f 2>&1 | tail -2; done
timeout 300 python tools/layer_bench.py 128 192 28 28 31 1 D8 f32 2>&1 | tail -2
timeout 600 python bench.py --model convnext_t_1d --steps 20 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-400
