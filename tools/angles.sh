#!/bin/bash
# per-angle forward/backward times at the stage-1 shape (all channels at one angle)
for a in 0 22.5 45 67.5 90 112.5 135 157.5; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-extra --no-e2e --no-cpu --angle $a "$@" 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('angle $a', round(d['value']), {k: round(v*1000,1) for k,v in d['per_pass_ms'].items()})"
done
