#!/bin/bash
# usage: tools/sweep.sh "PPC G" ...   (env O1D_PPC / O1D_G variants of the spec kernels)
for cfg in "$@"; do
  set -- $cfg
  O1D_PPC=$1 O1D_G=$2 timeout 300 python bench.py --steps 30 --warmup 5 --no-extra --no-e2e --no-cpu 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PPC=$1 G=$2', round(d['value']), {k: round(v*1000,1) for k,v in d['per_pass_ms'].items()}, d['plan'][:200])" 2>&1 | tail -1
done
