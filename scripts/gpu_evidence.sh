#!/bin/bash
# Round-2 evidence on one B200: op table, ncu --set full of every kernel on
# c3 (summarised to text on the box, reports deleted), the launch list of
# the bench, compute-sanitizer on a small run.
mkdir -p gpurun_out/ev
python scripts/prof_ops.py > gpurun_out/ev/prof_ops.json 2> gpurun_out/ev/prof_ops.err
K='regex:step_tma4_kernel|compact_count_kernel|compact_write_kernel|scatter_rows_kernel|stats_rows_vec_kernel|noise_kernel|aiu_rows_kernel|relocate_rows_kernel'
ncu --set full --clock-control none --import-source on -k "$K" --launch-count 30 -o /tmp/ops_full -f python scripts/prof_ops.py --reps 1 > gpurun_out/ev/ncu_ops.log 2>&1
python scripts/ncu_summary.py /tmp/ops_full.ncu-rep > gpurun_out/ev/ncu_ops_summary.txt 2>&1
ncu -i /tmp/ops_full.ncu-rep --page source --csv -k regex:step_tma4 --launch-count 1 > /tmp/src.csv 2>/dev/null; head -c 2000000 /tmp/src.csv > gpurun_out/ev/ncu_step_tma4_source_head.csv
rm -f /tmp/ops_full.ncu-rep
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/launches_c3.csv python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-legs > gpurun_out/ev/ncu_launches.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py > gpurun_out/ev/sanitizer_$tool.log 2>&1
  GS_FIXED_VARIANT=21 timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py > gpurun_out/ev/sanitizer_${tool}_ring.log 2>&1
done
for f in gpurun_out/ev/sanitizer_*.log; do echo "== $f"; tail -n 3 $f; done
du -sh gpurun_out
