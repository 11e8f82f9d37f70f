#!/bin/bash
# sparse masks: 3 CTAs per SM (3 scanning loaders per SM) vs the default 2
source scripts/gpu_iter_lib.sh
for lv in 0 1 2; do
  one c5_1_lv$lv "GS_TMA4_BW=1 GS_LOWVIS_SHAPE=$lv" --workload c5 --vis 0.01 --steps 20
  one c5_3_lv$lv "GS_TMA4_BW=1 GS_LOWVIS_SHAPE=$lv" --workload c5 --vis 0.03 --steps 20
  one 625_1_lv$lv "GS_TMA4_BW=1 GS_LOWVIS_SHAPE=$lv" --workload c5 --rows 6250000 --vis 0.01
done
one c5_10_lv0 "GS_TMA4_BW=1 GS_LOWVIS_SHAPE=0" --workload c5 --vis 0.1 --steps 10
one c5_10_lv1 "GS_TMA4_BW=1 GS_LOWVIS_SHAPE=1" --workload c5 --vis 0.1 --steps 10
