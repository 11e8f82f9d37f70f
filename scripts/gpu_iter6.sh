#!/bin/bash
# streaming fused kernel on big clouds: per-CTA mask slices vs tiles dealt grid-stride
source scripts/gpu_iter_lib.sh
for sl in 2 1; do
  one c3_s$sl GS_MASK_SLICES=$sl --workload c3
  one c3coh_s$sl "GS_MASK_SLICES=$sl" --workload c3 --mask coherent
  one 625_1_s$sl GS_MASK_SLICES=$sl --workload c5 --rows 6250000 --vis 0.01
  one 625_30_s$sl GS_MASK_SLICES=$sl --workload c5 --rows 6250000 --vis 0.3
  one c5_1_s$sl GS_MASK_SLICES=$sl --workload c5 --vis 0.01 --steps 20
  one c5_30_s$sl GS_MASK_SLICES=$sl --workload c5 --vis 0.3 --steps 10
  one c5_100_s$sl GS_MASK_SLICES=$sl --workload c5 --vis 1.0 --steps 10
done
