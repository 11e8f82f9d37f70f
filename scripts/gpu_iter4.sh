#!/bin/bash
# crossover: two-phase (bias warp) vs K1 + K2 (bias warp / loader-staged) by cloud size
source scripts/gpu_iter_lib.sh
for r in 50000 100000 200000 400000 800000; do
  one tp_$r "GS_TMA4_BW=1 GS_FUSED_MODE=2" --workload c1 --rows $r
  one idx1_$r "GS_TMA4_BW=1" --workload c1 --rows $r --no-fused
  one idx0_$r "GS_TMA4_BW=0" --workload c1 --rows $r --no-fused
done
one tp_c2 "GS_TMA4_BW=1 GS_FUSED_MODE=2" --workload c2
one idx1_c2 "GS_TMA4_BW=1" --workload c2 --no-fused
one tp_c4 "GS_TMA4_BW=1 GS_FUSED_MODE=2" --workload c4
one idx0_c4 "GS_TMA4_BW=0" --workload c4 --no-fused
one tp_c3_p10 "GS_TMA4_BW=1 GS_FUSED_MODE=2" --workload c3 --vis 0.1
one st_c3_p10 "X=1" --workload c3 --vis 0.1
one tp_1pct "GS_TMA4_BW=1 GS_FUSED_MODE=2" --workload c5 --rows 3000000 --vis 0.01
one st_1pct "X=1" --workload c5 --rows 3000000 --vis 0.01
one idx1_1pct "GS_TMA4_BW=1" --workload c5 --rows 3000000 --vis 0.01 --no-fused
