#!/bin/bash
# GPU tests + K2 timing for both parameter layouts (record vs per-attribute).
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
if [ -z "$NOTEST" ]; then
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
fi
for lay in ${LAYOUTS:-record attr}; do
  for m in ${MASKS:-bernoulli}; do
    python bench.py --params $lay --mask $m --no-e2e --no-cpu --steps 50 $BENCH_ARGS > gpurun_out/q_${lay}_$m.json 2>&1
    python -c "
import json; d=json.loads(open('gpurun_out/q_${lay}_$m.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$lay $m', round(d['value']/1e9,3),'G/s', round(d['ms_per_step'],4),'ms k2', round(r['k2_ms_avg'],4), 'frac', round(r['frac'],3), 'step_frac', round(r['step_frac'],3))" 2>&1 | tail -1
  done
done
if [ -n "$E2E" ]; then
  python bench.py --no-cpu --steps 20 > gpurun_out/e2e_record.json 2>&1; echo "e2e rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/e2e_record.json').read().strip().splitlines()[-1]); e=d['e2e']; print('e2e', round(e['ms_per_step'],2), 'ms', round(e['value']/1e6,1), 'M/s dense', round(e['dense_copy']['ms_per_step'],2))"
fi
