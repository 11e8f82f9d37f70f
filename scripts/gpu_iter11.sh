#!/bin/bash
# the first chunk of every CTA emitted early (GS_EARLY_FIRST=1)
source scripts/gpu_iter_lib.sh
for e in 0 1 0 1; do
  one s625_1_e$e GS_EARLY_FIRST=$e --workload c5 --rows 6250000 --vis 0.01
  one c5_1_e$e GS_EARLY_FIRST=$e --workload c5 --vis 0.01 --steps 20
  one c1_e$e GS_EARLY_FIRST=$e --workload c1
  one m1_3_e$e GS_EARLY_FIRST=$e --workload c5 --rows 1000000 --vis 0.03
done
