cd $GRAFT_REPO_ROOT
for cfg in "4 0" "16 0" "4 128" "16 128"; do set -- $cfg
for m in bernoulli coherent; do
GS_STATE_ROW_ALIGN=$2 python bench.py --record-align $1 --mask $m --no-e2e --no-cpu --steps 50 > gpurun_out/al.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/al.json').read().strip().splitlines()[-1]); r=d['roofline']; print('align $1 state $2 $m', round(d['ms_per_step'],4),'ms k2', round(r['k2_ms_avg'],4), 'frac', round(r['frac'],3))"
done; done
