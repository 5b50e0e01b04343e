#!/bin/bash
# pairs x slots per pair (O1D_P, O1D_NBUF) with on-demand claims, fp32 / bf16 S1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for cfg in "O1D_P=3 O1D_NBUF=3" "O1D_P=4 O1D_NBUF=2" "O1D_P=3 O1D_NBUF=3" "O1D_P=4 O1D_NBUF=2"; do
  env $cfg timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu --no-e2e --no-extra > gpurun_out/sl.json 2>&1; echo "$cfg f32 $(python tools/bench_brief.py gpurun_out/sl.json | cut -c1-200)"; python -c "import json; d=json.loads(open('gpurun_out/sl.json').read().strip().splitlines()[-1]); print('   ', d['plan'][60:330])"
done
