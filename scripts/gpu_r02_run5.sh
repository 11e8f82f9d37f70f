#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/pytest_gpu_full.log
cat gpurun_out/pytest_gpu_full.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3_full.json 2> gpurun_out/bench_c3_full.err
tail -c 300 gpurun_out/bench_c3_full.json
bash scripts/gpu_sweep_r02.sh
mkdir -p gpurun_out/ev
python scripts/prof_ops.py > gpurun_out/ev/prof_ops.json 2> gpurun_out/ev/prof_ops.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/ev/prof_ops.json"))
for k, v in d["ops"].items():
    print("%-62s %8.4f ms %7.0f GB/s frac %.3f %s" % (k, v["ms"], v["GB/s"], v["frac"], v["note"]))
PY
tail -3 gpurun_out/ev/prof_ops.err
