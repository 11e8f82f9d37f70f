#!/bin/bash
# GPU tests + K2 timing per (param layout, variant) pair.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
if [ -z "$NOTEST" ]; then
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
fi
for pv in ${PAIRS:-record:0 attr:0 attr:7}; do
  lay=${pv%%:*}; v=${pv##*:}
  for m in ${MASKS:-bernoulli coherent}; do
    GS_FIXED_VARIANT=$v timeout 300 python bench.py --params $lay --mask $m --no-e2e --no-cpu --steps 50 $BENCH_ARGS > gpurun_out/v.json 2>&1
    python -c "
import json; d=json.loads(open('gpurun_out/v.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$lay v$v $m', round(d['ms_per_step'],4),'ms k2', round(r['k2_ms_avg'],4), 'frac', round(r['frac'],3))" 2>&1 | tail -1
  done
done
