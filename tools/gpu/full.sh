TAG=${1:-x}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1; echo smoke rc $?
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -n 3 > gpurun_out/gpu_tests_$TAG.txt 2>&1; echo tests rc $?
tail -15 gpurun_out/gpu_tests_$TAG.txt
