#!/bin/bash
# K2 timing per fixed-kernel variant (GS_FIXED_VARIANT) on the c3 workload.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
if [ -z "$NOTEST" ]; then
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
fi
for v in ${VARIANTS:-0 8}; do
  for m in ${MASKS:-bernoulli}; do
    GS_FIXED_VARIANT=$v timeout 300 python bench.py --mask $m --no-e2e --no-cpu --steps 50 $BENCH_ARGS > gpurun_out/v_${v}_$m.json 2>&1
    python -c "
import json; d=json.loads(open('gpurun_out/v_${v}_$m.json').read().strip().splitlines()[-1]); r=d['roofline']; print('v$v $m', round(d['value']/1e9,3),'G/s', round(d['ms_per_step'],4),'ms k2', round(r['k2_ms_avg'],4), 'frac', round(r['frac'],3), 'step_frac', round(r['step_frac'],3))" 2>&1 | tail -1
  done
done
