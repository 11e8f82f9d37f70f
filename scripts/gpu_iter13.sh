#!/bin/bash
# dynamic tail size: GS_DYN_TAIL = eighths of the tiles claimed dynamically
source scripts/gpu_iter_lib.sh
for d in 0 1 2 0 1 2; do
  one s625_1_d$d GS_DYN_TAIL=$d --workload c5 --rows 6250000 --vis 0.01
  one c5_1_d$d GS_DYN_TAIL=$d --workload c5 --vis 0.01 --steps 20
  one c5_3_d$d GS_DYN_TAIL=$d --workload c5 --vis 0.03 --steps 20
  one c3_d$d GS_DYN_TAIL=$d --workload c3
done
