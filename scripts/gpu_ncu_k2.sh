#!/bin/bash
# ncu --set full of one K2 launch (the fused TMA step) on c3 for each
# GS_TMA4_BW setting, summarised on the box.
mkdir -p gpurun_out/ncu
for bw in 0 1; do
  GS_TMA4_BW=$bw ncu --set full --clock-control none --import-source on -k regex:step_tma4 --launch-skip 4 --launch-count 1 -o /tmp/k2_bw$bw -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-legs --no-graph > gpurun_out/ncu/k2_bw$bw.log 2>&1
  python scripts/ncu_summary.py /tmp/k2_bw$bw.ncu-rep --bytes 2995000000 > gpurun_out/ncu/k2_bw$bw.txt 2>&1
  ncu -i /tmp/k2_bw$bw.ncu-rep --page details --csv > gpurun_out/ncu/k2_bw${bw}_details.csv 2>&1
done
cat gpurun_out/ncu/k2_bw0.txt gpurun_out/ncu/k2_bw1.txt
