#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/pytest_gpu_full.log
python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
cat gpurun_out/pytest_gpu_full.log
python - <<'PY'
import json
for f in ["gpurun_out/bench_c3.json"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "FAILED", e); continue
    r = d["roofline"]
    print(f, "value %.4g ms %.4f K2 %.4f frac %.3f fused %s" % (d["value"], d["ms_per_step"], r["k2_ms_avg"], r["frac"], r.get("fused_compaction")))
    for k, v in (d.get("legs") or {}).items():
        print("  ", k, "%.4g ms %.4f frac %.3f step_frac %.3f" % (v["value"], v["ms_per_step"], v["roofline"]["frac"], v["roofline"]["step_frac"]))
    if d.get("e2e"): print("   e2e %.4g" % d["e2e"]["value"])
PY
tail -3 gpurun_out/bench_c3.err
bash scripts/gpu_evidence.sh
