python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1 | cut -c1-200
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "full_stage1 or angle_sets_spec or step_fused or assignments_spec or bf16" -n 3 2>&1 | tail -3
bash tools/ab_r2.sh "O1D_EARLY=0" "O1D_EARLY=1" "O1D_EARLY=0 O1D_PAIRMAP=1" "O1D_EARLY=1 O1D_PAIRMAP=1"
BENCH_ARGS="--dtype bf16" bash tools/ab_r2.sh "O1D_EARLY=0" "O1D_EARLY=1"
