mkdir -p gpurun_out profiles/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.txt 2>&1; echo smoke rc $?
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ffma2_bench tools/ffma2_bench.cu && /tmp/ffma2_bench > gpurun_out/ffma.txt 2>&1; cat gpurun_out/ffma.txt
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
tail -c 1500 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -n 3 > gpurun_out/gpu_tests.txt 2>&1; echo tests rc $?
tail -40 gpurun_out/gpu_tests.txt
