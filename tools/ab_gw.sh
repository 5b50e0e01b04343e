#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -n 3 -k "generic or tiny or block1d or stride2 or convnext or outputs_fully or bilinear or shear or ragged" 2>&1 | tail -1
for a in "128 64 224 224 5 2 0" "128 64 112 112 5 1 90" "128 64 112 112 5 2 90" "128 192 28 28 31 1 D8"; do timeout 300 python tools/layer_bench.py $a bf16 1 2>&1 | tail -1 | cut -c1-170; done
timeout 600 python bench.py --model convnext_t_1d --steps 20 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-200
