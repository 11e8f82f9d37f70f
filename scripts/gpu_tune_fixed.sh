#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for v in 0 1 2 3; do
  GS_FIXED_VARIANT=$v python bench.py --no-e2e --no-cpu --steps 50 > gpurun_out/tunef_v$v.json 2>&1; echo "fixed v$v rc=$?"
done
GS_FIXED_VARIANT=0 python bench.py --no-e2e --no-cpu --steps 50 --mask coherent > gpurun_out/tunef_coh.json 2>&1
for f in gpurun_out/tunef_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']; print('$f', round(d['value']/1e9,3),'G/s', round(d['ms_per_step'],3),'ms k2', round(r['k2_ms_avg'],4), 'frac', round(r['frac'],3))" 2>&1 | tail -1; done
