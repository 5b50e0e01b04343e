#!/bin/bash
# A/B of plan-time knobs at S1 (fp32 unless BENCH_ARGS says otherwise); prints step + per-pass us
# usage: bash tools/ab_r2.sh "ENV=.." "ENV=.. ENV2=.." ...
for cfg in "$@"; do
  env $cfg timeout 300 python bench.py --steps 100 --warmup 5 --no-extra --no-e2e --no-cpu $BENCH_ARGS > /tmp/o.json 2>/tmp/o.err
  python -c "import json,sys; d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); print('$cfg', round(d['value']), round(d['ms_per_step']*1000,1), {k: round(v*1000,1) for k,v in d['per_pass_ms'].items()}, d['plan'][-120:])" 2>/dev/null || tail -3 /tmp/o.err
done
