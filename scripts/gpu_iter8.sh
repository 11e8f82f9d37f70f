#!/bin/bash
# two-phase kernel after the phase-A prefetch
source scripts/gpu_iter_lib.sh
one tp_c1 GS_FUSED_MODE=2 --workload c1
one tp_c1coh GS_FUSED_MODE=2 --workload c1 --mask coherent
one c2 X=1 --workload c2
one tp_625_1 GS_FUSED_MODE=2 --workload c5 --rows 6250000 --vis 0.01
one st_625_1 X=1 --workload c5 --rows 6250000 --vis 0.01
one tp_3m_1 GS_FUSED_MODE=2 --workload c5 --rows 3000000 --vis 0.01
one st_3m_1 X=1 --workload c5 --rows 3000000 --vis 0.01
one tp_c3 GS_FUSED_MODE=2 --workload c3
