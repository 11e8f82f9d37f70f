#!/bin/bash
mkdir -p gpurun_out/ev
python -m pytest tests/test_gpu_api_r02.py -q -p no:cacheprovider -k "fused_compaction or tma_record" 2>&1 | tail -3
bash scripts/gpu_sweep_r02.sh
python scripts/prof_ops.py > gpurun_out/ev/prof_ops.json 2> gpurun_out/ev/prof_ops.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/ev/prof_ops.json"))
for k, v in d["ops"].items():
    print("%-62s %8.4f ms %7.0f GB/s frac %.3f %s" % (k, v["ms"], v["GB/s"], v["frac"], v["note"]))
PY
K='regex:step_tma4_kernel|compact_count_kernel|compact_write_kernel|scatter_rows_kernel|stats_rows_vec_kernel|noise_kernel|aiu_rows_kernel|relocate_rows_kernel|philox'
ncu --set full --clock-control none -k "$K" --launch-count 40 -o /tmp/ops_full -f python scripts/prof_ops.py --reps 1 > gpurun_out/ev/ncu_ops.log 2>&1
python scripts/ncu_summary.py /tmp/ops_full.ncu-rep > gpurun_out/ev/ncu_ops_summary.txt 2>&1
rm -f /tmp/ops_full.ncu-rep
grep -E "^kernel|duration|dram throughput|dram bytes total|issue active|top stalls" gpurun_out/ev/ncu_ops_summary.txt | head -120
