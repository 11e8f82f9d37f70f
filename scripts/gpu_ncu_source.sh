#!/bin/bash
# Source-level warp-stall sampling of the fused step kernel (ncu --set full
# --import-source on), summarised on the box: the hottest CUDA source lines.
# usage: gpu_ncu_source.sh <tag> <bench args...>
tag=$1; shift
mkdir -p gpurun_out/ncu_src
ncu --set full --import-source on --clock-control none -k regex:step_tma4 --launch-skip 6 --launch-count 1 \
  -o /tmp/src_$tag -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-legs --no-graph "$@" \
  > gpurun_out/ncu_src/$tag.log 2>&1
python scripts/ncu_summary.py /tmp/src_$tag.ncu-rep > gpurun_out/ncu_src/${tag}_summary.txt 2>&1
ncu -i /tmp/src_$tag.ncu-rep --page source --csv --print-source sass > /tmp/src_$tag.csv 2> gpurun_out/ncu_src/${tag}_src.err
python scripts/ncu_source_top.py /tmp/src_$tag.csv > gpurun_out/ncu_src/${tag}_hot_sass.txt 2>&1
head -c 1500 /tmp/src_$tag.csv > gpurun_out/ncu_src/${tag}_csv_head.txt
gzip -c /tmp/src_$tag.csv > gpurun_out/ncu_src/${tag}_sass.csv.gz
ncu -i /tmp/src_$tag.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src2_$tag.csv 2>/dev/null; gzip -c /tmp/src2_$tag.csv > gpurun_out/ncu_src/${tag}_cudasass.csv.gz
rm -f /tmp/src_$tag.ncu-rep
