#!/bin/bash
# K2 timing for parameter/gradient record alignment x moment-record alignment.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for cfg in ${CFGS:-"4 2" "16 2" "4 128" "16 128"}; do set -- $cfg
for m in bernoulli coherent; do
python bench.py --record-align $1 --state-align $2 --mask $m --no-e2e --no-cpu --steps 50 > gpurun_out/al.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/al.json').read().strip().splitlines()[-1]); r=d['roofline']; print('record-align $1 state-align $2 $m', round(d['ms_per_step'],4),'ms k2', round(r['k2_ms_avg'],4), 'frac', round(r['frac'],3))"
done; done
