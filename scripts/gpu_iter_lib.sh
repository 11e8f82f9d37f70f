#!/bin/bash
# two-phase vs streaming fused vs K1+K2 on small / low-visibility clouds
mkdir -p gpurun_out/small
one() {  # tag, env, args
  tag=$1; shift; envs=$1; shift
  env $envs python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e --no-legs "$@" > gpurun_out/small/$tag.json 2> gpurun_out/small/$tag.err
  python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/small/{tag}.json").read().strip().splitlines()[-1])
except Exception as e:
    print(tag, "FAILED", e); sys.exit(0)
r = d["roofline"]
print("%-26s nv %9.0f step %.4f ms  K %.4f ms  frac %.3f step_frac %.3f fused %s" % (tag, d["visible_per_step"], d["ms_per_step"], r["k2_ms_avg"], r["frac"], r["step_frac"], r.get("fused_compaction")))
PY
}
