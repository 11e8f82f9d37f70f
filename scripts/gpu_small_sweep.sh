#!/bin/bash
# small-work latency: per-step and dominant-kernel device time on small clouds
# (fit time = intercept + bytes / slope over the row sweep)
mkdir -p gpurun_out/small
run() {
  tag=$1; shift
  python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e --no-legs "$@" > gpurun_out/small/$tag.json 2> gpurun_out/small/$tag.err
  python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/small/{tag}.json").read().strip().splitlines()[-1])
except Exception as e:
    print(tag, "FAILED", e); sys.exit(0)
r = d["roofline"]
print("%-22s nv %9.0f step %.4f ms  K %.4f ms  frac %.3f step_frac %.3f fused %s" % (tag, d["visible_per_step"], d["ms_per_step"], r["k2_ms_avg"], r["frac"], r["step_frac"], r.get("fused_compaction")))
PY
}
if [ -n "$SMALL_ONLY" ]; then
  for t in $SMALL_ONLY; do run $t --workload c1 --rows $t "${@}"; done
  exit 0
fi
run floor --workload c1 --vis 0.0001 "$@"
run floor_nofused --workload c1 --vis 0.0001 --no-fused "$@"
for r in 20000 50000 100000 200000 400000 800000 1600000; do
  run r$r --workload c1 --rows $r --no-fused "$@"
done
