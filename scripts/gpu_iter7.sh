#!/bin/bash
# bias warp on the small-cloud streaming kernel
source scripts/gpu_iter_lib.sh
for r in 100000 400000 1600000 3000000; do
  one st_bw0_$r GS_TMA4_BW=0 --workload c1 --rows $r
  one st_bw1_$r GS_TMA4_BW=1 --workload c1 --rows $r
done
one c4_bw0 GS_TMA4_BW=0 --workload c4
one c4_bw1 GS_TMA4_BW=1 --workload c4
