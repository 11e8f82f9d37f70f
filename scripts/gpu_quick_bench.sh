#!/bin/bash
# quick K2 check: c3 default line (no e2e / cpu) with the c5 legs
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e "$@" > gpurun_out/qb.json 2> gpurun_out/qb.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/qb.json").read().strip().splitlines()[-1])
r = d["roofline"]
print("value %.4g ms %.4f timed %.4f K %.4f frac %.3f fused %s" % (d["value"], d["ms_per_step"], d["ms_per_step_timed"], r["k2_ms_avg"], r["frac"], r.get("fused_compaction")))
for k, v in (d.get("legs") or {}).items():
    print("  ", k, "%.4g ms %.4f frac %.3f step_frac %.3f" % (v["value"], v["ms_per_step"], v["roofline"]["frac"], v["roofline"]["step_frac"]))
PY
tail -2 gpurun_out/qb.err
