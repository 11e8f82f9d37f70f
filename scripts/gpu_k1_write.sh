# A/B of the K1 write pass (profiles/r01/k1_persistent_write_ab.txt). The
# GS_COMPACT_WRITE switch lived in an experimental gs_compact.cu that was not
# adopted; with the committed kernel every variant runs the stock write pass.
cd $GRAFT_REPO_ROOT
for v in 0 1 2; do
  GS_COMPACT_WRITE=$v timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k compaction > gpurun_out/k1_t$v.log 2>&1; echo "tests v$v: $(tail -1 gpurun_out/k1_t$v.log)"
done
for rep in 1 2; do for v in 0 1 2; do
  GS_COMPACT_WRITE=$v timeout 600 python bench.py --workload c5 --vis 0.01 --no-e2e --no-cpu --steps 20 --warmup 3 > gpurun_out/k1_c5_$v.json 2>/dev/null
  GS_COMPACT_WRITE=$v timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/k1_c3_$v.json 2>/dev/null
  python -c "
import json
for w in ('c5','c3'):
    d=json.loads(open('gpurun_out/k1_'+w+'_$v.json').read().strip().splitlines()[-1]); r=d['roofline']
    print('v$v', w, round(d['ms_per_step'],4), 'k2', round(r['k2_ms_avg'],4), 'step_frac', round(r['step_frac'],3))"
done; done
