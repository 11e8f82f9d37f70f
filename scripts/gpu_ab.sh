#!/bin/bash
# A/B of two source trees on the same box: .ab/old (a git archive) against HEAD
set -e
(cd .ab/old && python -m paper_2601_16736_b200._build > /dev/null 2>&1)
source scripts/gpu_iter_lib.sh
oldone() {  # tag, args
  tag=$1; shift
  (cd .ab/old && python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e --no-legs "$@" 2>/dev/null | tail -1) > gpurun_out/small/$tag.json
  python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
d = json.loads(open(f"gpurun_out/small/{tag}.json").read().strip().splitlines()[-1])
r = d["roofline"]
print("%-26s nv %9.0f step %.4f ms  K %.4f ms  frac %.3f fused %s" % (tag, d["visible_per_step"], d["ms_per_step"], r["k2_ms_avg"], r["frac"], r.get("fused_compaction")))
PY
}
for rep in 1 2; do
  oldone old_c5_1 --workload c5 --vis 0.01 --steps 20
  one new_c5_1 X=1 --workload c5 --vis 0.01 --steps 20
  oldone old_625_1 --workload c5 --rows 6250000 --vis 0.01
  one new_625_1 X=1 --workload c5 --rows 6250000 --vis 0.01
  oldone old_c3 --workload c3
  one new_c3 X=1 --workload c3
done
