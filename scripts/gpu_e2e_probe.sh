#!/bin/bash
# e2e zero-copy probe: record gradients through L1 (.ca) vs L2-only (.cg), and per-attribute.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for v in "record 1" "record 0" "attr x"; do
  set -- $v
  if [ "$2" = x ]; then unset GS_GREC_CA; else export GS_GREC_CA=$2; fi; python bench.py --no-cpu --steps 10 --params $1 > gpurun_out/e2e_$1_$2.json 2>&1; echo "$v rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/e2e_$1_$2.json').read().strip().splitlines()[-1]); e=d['e2e']; print('$v', 'k2', round(d['roofline']['k2_ms_avg'],4), 'e2e', round(e['ms_per_step'],2), 'ms', round(e['value']/1e6,1), 'M/s dense', round(e['dense_copy']['ms_per_step'],2))"
done
