#!/bin/bash
# ncu --set full of the generic kernels at the ConvNeXt stem shapes (bf16): 112^2 s1 90 deg, 224^2 s2 0 deg
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:generic -s 3 -c 3 -o gpurun_out/full_generic112 \
    python tools/layer_bench.py 32 64 112 112 5 1 90 bf16 > /dev/null 2>&1; echo rc $?
ncu --set full --clock-control none --import-source on -k regex:"generic|strided" -s 4 -c 4 -o gpurun_out/full_generic224 \
    python tools/layer_bench.py 32 64 224 224 5 2 0 bf16 > /dev/null 2>&1; echo rc $?
python tools/ncu_summary.py gpurun_out/full_generic112.ncu-rep > gpurun_out/ncu_generic112_summary.txt 2>&1
python tools/ncu_summary.py gpurun_out/full_generic224.ncu-rep > gpurun_out/ncu_generic224_summary.txt 2>&1
cat gpurun_out/ncu_generic112_summary.txt gpurun_out/ncu_generic224_summary.txt
