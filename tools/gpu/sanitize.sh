python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
mkdir -p gpurun_out
for tool in memcheck racecheck initcheck synccheck; do
  echo "== compute-sanitizer --tool $tool (tools/sanitize_cases.py)"
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py 2>&1 | grep -v "^$" | tail -14
  echo "rc=$?"
done > gpurun_out/sanitizer_r2.txt 2>&1
cat gpurun_out/sanitizer_r2.txt
