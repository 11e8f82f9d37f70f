#!/bin/bash
# Round-2 evidence on one B200: the op table (prof_ops.py), one ncu --set
# full capture per kernel family on c3 (summarised on the box, reports
# deleted), and the ncu launch list of the bench command.  compute-sanitizer
# is closed on this pool (it left GPUs needing a reset); not run.
mkdir -p gpurun_out/ev
python scripts/prof_ops.py > gpurun_out/ev/prof_ops.json 2> gpurun_out/ev/prof_ops.err
for k in step_tma4_kernel compact_count_kernel compact_write_kernel scatter_rows_kernel stats_rows_vec_kernel noise_rec_kernel aiu_rows_kernel relocate_rows_kernel philox_bernoulli_kernel; do
  ncu --set full --clock-control none -k regex:$k --launch-count 1 -o /tmp/ev_$k -f python scripts/prof_ops.py --reps 1 > gpurun_out/ev/ncu_$k.log 2>&1
  python scripts/ncu_summary.py /tmp/ev_$k.ncu-rep > gpurun_out/ev/ncu_$k.txt 2>&1
  rm -f /tmp/ev_$k.ncu-rep
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/launches_c3.csv python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-legs > gpurun_out/ev/ncu_launches.log 2>&1
cat gpurun_out/ev/ncu_*.txt | grep -E "^kernel|duration|dram throughput|dram bytes total|issue active|occupancy|top stalls"
