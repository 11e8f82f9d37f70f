#!/bin/bash
# e2e (zero-copy host gradients) per K2 variant / gradient-copy policy.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for cfg in "0 1" "0 0" "9 0" "10 0" "12 0" "11 0"; do
  set -- $cfg
  GS_FIXED_VARIANT=$1 GS_GREC_CA=$2 timeout 300 python bench.py --no-cpu --steps 20 > gpurun_out/e2e_v$1_ca$2.json 2> gpurun_out/e2e_v$1_ca$2.err
  python -c "
import json; d=json.loads(open('gpurun_out/e2e_v$1_ca$2.json').read().strip().splitlines()[-1]); e=d['e2e']; print('v$1 ca$2 k2', round(d['roofline']['k2_ms_avg'],4), 'e2e ms', round(e['ms_per_step'],3), 'G/s', round(e['value']/1e9,4))" 2>&1 | tail -1
done
