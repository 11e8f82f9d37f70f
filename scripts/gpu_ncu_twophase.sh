#!/bin/bash
# ncu --set full of the two-phase fused kernel (c2: 1M rows, coupled sparse-adam)
mkdir -p gpurun_out/ncu_tp
ncu --set full --clock-control none -k regex:step_tma4 --launch-skip 8 --launch-count 1 \
  -o /tmp/tp_c2 -f python bench.py --workload c2 --steps 3 --warmup 3 --no-e2e --no-cpu --no-legs \
  > gpurun_out/ncu_tp/c2.log 2>&1
python scripts/ncu_summary.py /tmp/tp_c2.ncu-rep > gpurun_out/ncu_tp/ncu_step_tma4_twophase_c2.txt 2>&1
rm -f /tmp/tp_c2.ncu-rep
cat gpurun_out/ncu_tp/ncu_step_tma4_twophase_c2.txt
