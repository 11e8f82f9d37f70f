#!/bin/bash
# bias-warp loader (GS_TMA4_BW=1) vs loader-staged bias factors, index path and two-phase
source scripts/gpu_iter_lib.sh
for bw in 0 1; do
  one idx_c1_bw$bw GS_TMA4_BW=$bw --workload c1 --no-fused
  one idx_c2_bw$bw GS_TMA4_BW=$bw --workload c2 --no-fused
  one idx_c3_bw$bw GS_TMA4_BW=$bw --workload c3 --no-fused
  one idx_c3coh_bw$bw GS_TMA4_BW=$bw --workload c3 --no-fused --mask coherent
  one idx_1pct_bw$bw GS_TMA4_BW=$bw --workload c5 --rows 6250000 --vis 0.01 --no-fused
  one tp_c1_bw$bw "GS_TMA4_BW=$bw GS_FUSED_MODE=2" --workload c1
  one tp_1pct_bw$bw "GS_TMA4_BW=$bw GS_FUSED_MODE=2" --workload c5 --rows 6250000 --vis 0.01
  one tp_c3_bw$bw "GS_TMA4_BW=$bw GS_FUSED_MODE=2" --workload c3
done
