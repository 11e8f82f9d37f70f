#!/bin/bash
# dynamic tail of the streaming kernel's tile dealing (GS_DYN_TAIL=1)
source scripts/gpu_iter_lib.sh
for d in 0 1 0 1; do
  one s625_1_d$d GS_DYN_TAIL=$d --workload c5 --rows 6250000 --vis 0.01
  one c5_1_d$d GS_DYN_TAIL=$d --workload c5 --vis 0.01 --steps 20
  one c5_3_d$d GS_DYN_TAIL=$d --workload c5 --vis 0.03 --steps 20
done
one c3_d0 GS_DYN_TAIL=0 --workload c3
one c3_d1 GS_DYN_TAIL=1 --workload c3
one s625_30_d0 GS_DYN_TAIL=0 --workload c5 --rows 6250000 --vis 0.3
one s625_30_d1 GS_DYN_TAIL=1 --workload c5 --rows 6250000 --vis 0.3
