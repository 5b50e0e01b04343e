python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for sel in generic spec; do for tool in initcheck racecheck; do
  echo "== $tool $sel"; timeout 900 compute-sanitizer --tool $tool --print-limit 1 python tools/sanitize_cases.py $sel 2>&1 | grep -E "SUMMARY|^ok|Uninitialized|Race reported|at o1d|at void" | head -8
done; done
