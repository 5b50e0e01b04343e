python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 compute-sanitizer --tool initcheck --print-limit 3 python tools/sanitize_cases.py 2>&1 | head -60
timeout 900 compute-sanitizer --tool racecheck --print-limit 4 python tools/sanitize_cases.py 2>&1 | grep -v "^=========     and Read" | head -60
