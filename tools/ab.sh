#!/bin/bash
# A/B a list of env settings: tools/ab.sh "bench args" "ENV=.. ENV2=.." "..."
# prints value / per-pass us / plan registers for each env setting
args=$1; shift
for cfg in "$@"; do
  env $cfg timeout 300 python bench.py --no-extra --no-e2e --no-cpu --steps 100 $args > /tmp/o.json 2>&1
  python -c "import json,sys; d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); import re; print('[$args] $cfg', round(d['value']), {k: round(v*1000,1) for k,v in d['per_pass_ms'].items()}, re.findall(r'Used \d+ registers', d.get('plan','')))" 2>/dev/null || { echo "[$args] $cfg FAILED"; tail -3 /tmp/o.json; }
done
