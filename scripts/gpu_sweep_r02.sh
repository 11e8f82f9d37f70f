#!/bin/bash
# Workload sweep on one B200: c1, c2, c4, c3 coherent / attr, c5 visibility
mkdir -p gpurun_out/sweep
run() {  # label, args
  local label=$1; shift
  python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-legs "$@" 2>/dev/null | tail -1 > gpurun_out/sweep/$label.json
  python - "$label" <<'PY'
import json, sys
lab = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/sweep/{lab}.json").read())
except Exception as e:
    print(lab, "FAILED", e); sys.exit()
r = d["roofline"]
print("%-22s step %.4f ms  value %.4g/s  K %.4f ms  frac %.3f  step_frac %.3f  fused %s" % (
    lab, d["ms_per_step"], d["value"], r["k2_ms_avg"], r["frac"], r["step_frac"], r.get("fused_compaction")))
PY
}
run c1 --workload c1
run c2 --workload c2
run c4 --workload c4
run c3_coherent --mask coherent
run c3_attr --params attr

for v in 0.01 0.03 0.1 0.3 1.0; do run c5_$v --workload c5 --vis $v --steps 10 --warmup 3; done
