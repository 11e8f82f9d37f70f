#!/bin/bash
# small clouds: streaming fused kernel with per-CTA mask slices vs two-phase vs K1 + K2
source scripts/gpu_iter_lib.sh
for r in 20000 100000 200000 400000 800000; do
  one st_$r GS_FUSED_MODE=1 --workload c1 --rows $r
  one tp_$r GS_FUSED_MODE=2 --workload c1 --rows $r
done
one st_c2 GS_FUSED_MODE=1 --workload c2
one tp_c2 GS_FUSED_MODE=2 --workload c2
one st_c4 GS_FUSED_MODE=1 --workload c4
one tp_c4 GS_FUSED_MODE=2 --workload c4
one st_3m1 GS_FUSED_MODE=1 --workload c5 --rows 3000000 --vis 0.01
one tp_3m1 GS_FUSED_MODE=2 --workload c5 --rows 3000000 --vis 0.01
one st_625_1 GS_FUSED_MODE=1 --workload c5 --rows 6250000 --vis 0.01
one st_c1_coh GS_FUSED_MODE=1 --workload c1 --mask coherent
one tp_c1_coh GS_FUSED_MODE=2 --workload c1 --mask coherent
