#!/bin/bash
# quick A/B: tools/quick.sh "ENV=.. ENV2=.." "..." -- prints value / per-pass ms for each env setting
for cfg in "$@"; do
  env $cfg timeout 300 python bench.py --no-extra --no-e2e --no-cpu > /tmp/o.json 2>&1
  python -c "import json,sys; d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); print('$cfg', round(d['value']), round(d['ms_per_step']*1000,1), {k: round(v*1000,1) for k,v in d['per_pass_ms'].items()})" 2>/dev/null || tail -3 /tmp/o.json
done
