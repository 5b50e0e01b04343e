# Round-2 GPU check: smoke, the -m gpu suite (3 workers), default bench line.
# usage (under gpurun): bash tools/gpu_check.sh TAG [extra bench args]
TAG=${1:-x}; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1; echo smoke rc $?; tail -2 gpurun_out/smoke_$TAG.txt
timeout 900 python bench.py --steps 100 --warmup 5 --no-cpu "$@" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc $?
python tools/bench_brief.py gpurun_out/bench_$TAG.json || tail -5 gpurun_out/bench_$TAG.err
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -n 3 > gpurun_out/gpu_tests_$TAG.txt 2>&1; echo tests rc $?
tail -15 gpurun_out/gpu_tests_$TAG.txt
