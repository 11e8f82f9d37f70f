# K1 count pass, two tiles per round: compaction parity, then c5 1% / c3 timing.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/k1c_t.log 2>&1; echo "tests: $(tail -1 gpurun_out/k1c_t.log)"
for rep in 1 2; do
  timeout 600 python bench.py --workload c5 --vis 0.01 --no-e2e --no-cpu --steps 20 --warmup 3 > gpurun_out/k1c_c5.json 2>/dev/null
  timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/k1c_c3.json 2>/dev/null
  python -c "
import json
for w in ('c5','c3'):
    d=json.loads(open('gpurun_out/k1c_'+w+'.json').read().strip().splitlines()[-1]); r=d['roofline']
    print('2tile', w, round(d['ms_per_step'],4), 'k2', round(r['k2_ms_avg'],4), 'step_frac', round(r['step_frac'],3))"
done
