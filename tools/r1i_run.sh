mkdir -p gpurun_out
bash tools/ab.sh "" "X=0" "O1D_P=5 O1D_NBUF=1" "O1D_P=6 O1D_NBUF=1" "O1D_P=5 O1D_NBUF=1 O1D_NPROD=1" > gpurun_out/ab_occ.txt 2>&1
timeout 1500 bash tools/profile_round.sh r1i > gpurun_out/profile_r1i.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_r1i.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r1i.txt 2>&1
tail -2 gpurun_out/gpu_tests_r1i.txt; cat gpurun_out/smoke_r1i.txt | tail -2
