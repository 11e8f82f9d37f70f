#!/bin/bash
# per-launch kernel durations (ncu, serialised) on small clouds, to split the
# graph-timed per-launch time into kernel duration and launch gap
mkdir -p gpurun_out/small_ncu
for cfg in "floor --vis 0.0001" "c1" "r400000 --rows 400000"; do
  set -- $cfg; tag=$1; shift
  ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg --clock-control none -c 120 --csv \
    --log-file gpurun_out/small_ncu/$tag.csv python bench.py --workload c1 --no-fused "$@" \
    --steps 8 --warmup 3 --no-cpu --no-e2e --no-legs > gpurun_out/small_ncu/$tag.log 2>&1
  python - $tag <<'PY'
import csv, sys, collections
tag = sys.argv[1]
rows = list(csv.reader(l for l in open(f"gpurun_out/small_ncu/{tag}.csv") if l.startswith('"')))
h = rows[0]; ki = h.index("Kernel Name"); mi = h.index("Metric Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit")
d = collections.defaultdict(list)
for r in rows[1:]:
    if r[mi] == "gpu__time_duration.sum":
        v = float(r[vi].replace(",", "")); v = v / 1000 if r[ui] == "nsecond" else v if r[ui] == "usecond" else v * 1000
        d[r[ki].split("(")[0][:60]].append(v)
for k, v in d.items():
    v = sorted(v)
    print(f"{tag:8s} {k:60s} n={len(v):3d} median {v[len(v)//2]:8.2f} us  min {v[0]:8.2f}")
PY
done
