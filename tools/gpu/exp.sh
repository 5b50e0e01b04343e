python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
bash tools/ab_r2.sh "O1D_P=4" "O1D_P=3 O1D_NBUF=3" "O1D_P=2 O1D_NBUF=4"
