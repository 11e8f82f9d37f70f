#!/bin/bash
# dynamic tail with block claims (GS_DYN_BLOCK tiles per atomic)
source scripts/gpu_iter_lib.sh
for rep in 1 2; do
  one c5_1_off "GS_DYN_TAIL=0" --workload c5 --vis 0.01 --steps 20
  one c5_1_b1 "GS_DYN_TAIL=1 GS_DYN_BLOCK=1" --workload c5 --vis 0.01 --steps 20
  one c5_1_b4 "GS_DYN_TAIL=1 GS_DYN_BLOCK=4" --workload c5 --vis 0.01 --steps 20
  one c5_1_b8 "GS_DYN_TAIL=2 GS_DYN_BLOCK=8" --workload c5 --vis 0.01 --steps 20
  one s625_off "GS_DYN_TAIL=0" --workload c5 --rows 6250000 --vis 0.01
  one s625_b4 "GS_DYN_TAIL=1 GS_DYN_BLOCK=4" --workload c5 --rows 6250000 --vis 0.01
  one c5_3_b1 "GS_DYN_BLOCK=1" --workload c5 --vis 0.03 --steps 20
  one c5_3_b4 "GS_DYN_BLOCK=4" --workload c5 --vis 0.03 --steps 20
  one c3_b1 "GS_DYN_BLOCK=1" --workload c3
  one c3_b2 "GS_DYN_BLOCK=2" --workload c3
done
