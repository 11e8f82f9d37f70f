#!/bin/bash
# ncu --set full of the fused step on small work (final build): c1 (per-CTA
# mask slices) and the 8-GPU shard of c5 at 1% (tiles grid-stride, bias warp)
mkdir -p gpurun_out/ncu_small_final
run() {  # tag, bench args
  tag=$1; shift
  ncu --set full --clock-control none -k regex:step_tma4 --launch-skip 8 --launch-count 1 \
    -o /tmp/ns_$tag -f python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-legs "$@" \
    > gpurun_out/ncu_small_final/$tag.log 2>&1
  python scripts/ncu_summary.py /tmp/ns_$tag.ncu-rep > gpurun_out/ncu_small_final/ncu_step_tma4_$tag.txt 2>&1
  rm -f /tmp/ns_$tag.ncu-rep
}
run c1 --workload c1
run shard8_1pct --workload c5 --rows 6250000 --vis 0.01
run c5_1pct --workload c5 --vis 0.01
cat gpurun_out/ncu_small_final/*.txt
