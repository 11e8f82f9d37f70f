#!/bin/bash
# Round-2 evidence on one B200: op table, ncu --set full of every kernel on
# c3, the launch list of the bench, sanitizers on a small run.
mkdir -p gpurun_out
python scripts/prof_ops.py > gpurun_out/prof_ops.json 2> gpurun_out/prof_ops.err
# ncu full captures, one launch of each kernel (after warm-up launches)
ncu --set full --clock-control none --import-source on -k regex:"step_tma4_kernel|compact_count_kernel|compact_write_kernel|scatter_rows_kernel|stats_rows_vec_kernel|noise_kernel|aiu_rows_kernel|relocate_rows_kernel" --launch-skip 0 --launch-count 40 -o gpurun_out/ops_full -f python scripts/prof_ops.py --reps 1 > gpurun_out/ncu_ops.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-legs > gpurun_out/ncu_launches.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitizer_$tool.log 2>&1
  GS_FIXED_VARIANT=21 timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitizer_${tool}_ring.log 2>&1
done
tail -3 gpurun_out/sanitizer_*.log
cat gpurun_out/prof_ops.json
