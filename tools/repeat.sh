#!/bin/bash
# repeat a bench configuration: tools/repeat.sh N [bench args...]
n=$1; shift
for i in $(seq $n); do
  timeout 300 python bench.py --no-extra --no-e2e --no-cpu --steps 100 "$@" > /tmp/o.json 2>&1
  python -c "import json; d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); print('$*', round(d['value']), {k: round(v*1000,1) for k,v in d['per_pass_ms'].items()}, d['clocks']['sm_mhz'])" 2>/dev/null || tail -3 /tmp/o.json
done
