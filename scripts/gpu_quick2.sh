#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for w in ${WORKLOADS:-c3 c1}; do
  python bench.py --workload $w --no-e2e --no-cpu --steps 50 $BENCH_ARGS > gpurun_out/q_$w.json 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/q_$w.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$w', round(d['value']/1e9,3),'G/s', round(d['ms_per_step'],4),'ms k2', round(r['k2_ms_avg'],4), 'frac', round(r['frac'],3), 'step_frac', round(r['step_frac'],3))" 2>&1 | tail -1
done
if [ -n "$LAUNCHES" ]; then
  CMD="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu"
  $CMD > gpurun_out/plain_short.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
fi
