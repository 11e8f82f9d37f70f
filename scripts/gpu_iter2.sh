#!/bin/bash
# two-phase vs streaming fused vs K1+K2 on small / low-visibility clouds
source scripts/gpu_iter_lib.sh
for r in 20000 100000 400000 1600000; do
  one tp_$r GS_FUSED_MODE=2 --workload c1 --rows $r
  one idx_$r X=1 --workload c1 --rows $r --no-fused
done
one floor_tp GS_FUSED_MODE=2 --workload c1 --vis 0.0001
one s1pct_tp GS_FUSED_MODE=2 --workload c5 --rows 6250000 --vis 0.01
one s1pct_stream GS_FUSED_MODE=1 --workload c5 --rows 6250000 --vis 0.01
one s1pct_idx X=1 --workload c5 --rows 6250000 --vis 0.01 --no-fused
one c2_tp GS_FUSED_MODE=2 --workload c2
one c2_idx X=1 --workload c2 --no-fused
one c3_tp GS_FUSED_MODE=2 --workload c3
one c3_stream X=1 --workload c3
