mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.txt 2>&1; echo smoke rc $?
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:randomly > gpurun_out/gpu_tests.txt 2>&1; echo tests rc $?
tail -30 gpurun_out/gpu_tests.txt
timeout 600 python bench.py --steps 50 --warmup 5 --no-extra --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
tail -c 3000 gpurun_out/bench.json
