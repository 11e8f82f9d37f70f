#!/bin/bash
# K2 shape sweep of the 2-D TMA record kernel (GS_TMA4_SHAPE) on c3, plus the
# cp.async ring (GS_FIXED_VARIANT=21) for reference.  One B200.
mkdir -p gpurun_out
out=gpurun_out/tma4_sweep.txt
: > $out
run() {  # label, env, args
  local label=$1; shift
  local envs=$1; shift
  env $envs python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e "$@" 2>/dev/null | tail -1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('%-34s step %.4f ms  K2 %.4f ms  frac %.3f' % ('$label', d['ms_per_step'], r['k2_ms_avg'], r['frac']))" >> $out
}
for sh in 0 1 2 3 4 5; do run "c3 tma4 shape $sh" "GS_TMA4_SHAPE=$sh"; done
run "c3 ring (variant 21)" "GS_FIXED_VARIANT=21"
for sh in 0 1; do run "c3 coherent tma4 shape $sh" "GS_TMA4_SHAPE=$sh" --mask coherent; done
run "c3 coherent ring" "GS_FIXED_VARIANT=21" --mask coherent
for sh in 0 1; do run "c5 100% tma4 shape $sh" "GS_TMA4_SHAPE=$sh" --workload c5 --vis 1.0 --steps 5 --warmup 3; done
run "c5 100% ring" "GS_FIXED_VARIANT=21" --workload c5 --vis 1.0 --steps 5 --warmup 3
cat $out
