#!/bin/bash
# c5: 50M SH-3 Gaussians on one B200, visibility sweep 1%..100% (K2 roofline per point).
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for v in ${VIS:-0.01 0.1 0.3 1.0}; do
  timeout 600 python bench.py --workload c5 --vis $v --no-e2e --no-cpu --steps 20 --warmup 3 > gpurun_out/c5_$v.json 2> gpurun_out/c5_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/c5_$v.json').read().strip().splitlines()[-1]); r=d['roofline']; print('c5 vis $v', round(d['value']/1e9,3),'G/s', round(d['ms_per_step'],4),'ms k2', round(r['k2_ms_avg'],4), 'frac', round(r['frac'],3), 'step_frac', round(r['step_frac'],3))" 2>&1 | tail -1
done
