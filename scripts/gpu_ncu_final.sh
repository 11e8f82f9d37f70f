#!/bin/bash
# ncu --set full of the default fused step on c3 as the bench runs it (CUDA
# graph replays, layout hints set by the warm-up steps), summarised on the box
mkdir -p gpurun_out/ncu_final
ncu --set full --clock-control none --import-source on -k regex:step_tma4 --launch-skip 6 --launch-count 1 \
  -o /tmp/k2c3 -f python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-legs > gpurun_out/ncu_final/c3.log 2>&1
python scripts/ncu_summary.py /tmp/k2c3.ncu-rep --bytes 2993600000 > gpurun_out/ncu_final/ncu_step_tma4_kernel_c3.txt 2>&1
ncu -i /tmp/k2c3.ncu-rep --page details --csv > gpurun_out/ncu_final/c3_details.csv 2>&1
ncu -i /tmp/k2c3.ncu-rep --page source --csv --print-source cuda,sass > /tmp/k2c3_src.csv 2>/dev/null
python scripts/ncu_cuda_lines.py /tmp/k2c3_src.csv 30 > gpurun_out/ncu_final/c3_hot_lines.txt 2>&1
rm -f /tmp/k2c3.ncu-rep
cat gpurun_out/ncu_final/ncu_step_tma4_kernel_c3.txt
