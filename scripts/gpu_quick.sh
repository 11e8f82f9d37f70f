#!/bin/bash
# Quick loop: GPU tests (parity) + K2 timing over the fixed-kernel variants + one ncu of the default.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for v in ${VARIANTS:-0 1 2 3}; do
  GS_FIXED_VARIANT=$v python bench.py --no-e2e --no-cpu --steps 50 > gpurun_out/q_v$v.json 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/q_v$v.json').read().strip().splitlines()[-1]); r=d['roofline']; print('v$v', round(d['value']/1e9,3),'G/s', round(d['ms_per_step'],3),'ms k2', round(r['k2_ms_avg'],4), 'frac', round(r['frac'],3))" 2>&1 | tail -1
done
if [ -n "$PROF" ]; then GS_FIXED_VARIANT=$PROF bash scripts/gpu_prof.sh q step_fixed_kernel; fi
