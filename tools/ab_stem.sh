#!/bin/bash
# generic-kernel change check: stride-2 parity (tiny / angle sets / block1d / shear / bilinear) + the stem layer timings
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -n 3 -k "tiny or angle_sets or block1d or shear_disc or bilinear or ragged or full_stage1_stride2" 2>&1 | tail -2
for a in "128 64 224 224 5 2 0" "128 64 112 112 5 1 90" "128 64 112 112 5 2 90"; do timeout 300 python tools/layer_bench.py $a bf16 2>&1 | tail -1 | cut -c1-170; done
timeout 600 python bench.py --model convnext_t_1d --steps 20 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-330
