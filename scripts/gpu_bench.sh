#!/bin/bash
# Bench + ncu evidence on one B200 (run under gpurun from the repo root).
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench rc=$?"
python bench.py --mask coherent --no-cpu --no-e2e > gpurun_out/bench_c3_coherent.json 2>&1; echo "coherent rc=$?"
python bench.py --params attr --no-cpu --no-e2e > gpurun_out/bench_c3_attr.json 2>&1; echo "attr rc=$?"
for w in c1 c2 c4; do
  python bench.py --workload $w --no-cpu --no-e2e > gpurun_out/bench_$w.json 2>&1; echo "$w rc=$?"
done
CMD="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu"
$CMD > gpurun_out/plain_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:step_ring_kernel -s 2 -c 1 -o gpurun_out/prof_step $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
python scripts/ncu_summary.py gpurun_out/prof_step.ncu-rep --bytes 2995021752 > gpurun_out/ncu_step_summary.txt 2>&1
tail -c 3000 gpurun_out/bench_c3.json
