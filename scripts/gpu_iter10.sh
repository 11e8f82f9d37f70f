#!/bin/bash
# dense masks at 3 CTAs per SM (measurement shapes 3 / 4)
source scripts/gpu_iter_lib.sh
for lv in -1 3 4; do
  one c3_lv$lv "GS_LOWVIS_SHAPE=$lv" --workload c3
  one c5_30_lv$lv "GS_LOWVIS_SHAPE=$lv" --workload c5 --vis 0.3 --steps 10
  one c5_10_lv$lv "GS_LOWVIS_SHAPE=$lv" --workload c5 --vis 0.1 --steps 10
done
