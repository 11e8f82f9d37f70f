#!/bin/bash
# ncu of the step kernel on small per-launch work: the 8-GPU shard of c5 at
# 1% (6.25M rows, fused) and c1 (100k rows, index path)
mkdir -p gpurun_out/ncu_small
ncu --set full --clock-control none -k regex:step_tma4 --launch-skip 6 --launch-count 1 -o /tmp/s1 -f python bench.py --workload c5 --rows 6250000 --vis 0.01 --steps 2 --warmup 3 --no-e2e --no-cpu --no-legs --no-graph > gpurun_out/ncu_small/s1.log 2>&1
python scripts/ncu_summary.py /tmp/s1.ncu-rep > gpurun_out/ncu_small/c5_shard8_1pct.txt 2>&1
ncu -i /tmp/s1.ncu-rep --page details --csv > gpurun_out/ncu_small/c5_shard8_1pct_details.csv 2>&1
ncu --set full --clock-control none -k regex:step_tma4 --launch-skip 20 --launch-count 1 -o /tmp/s2 -f python bench.py --workload c1 --steps 2 --warmup 3 --no-e2e --no-cpu --no-legs --no-graph > gpurun_out/ncu_small/s2.log 2>&1
python scripts/ncu_summary.py /tmp/s2.ncu-rep > gpurun_out/ncu_small/c1.txt 2>&1
ncu -i /tmp/s2.ncu-rep --page details --csv > gpurun_out/ncu_small/c1_details.csv 2>&1
cat gpurun_out/ncu_small/*.txt
