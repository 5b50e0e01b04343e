python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "stride or generic or ragged or tiny or bilinear or shear" -n 3 2>&1 | tail -4
