#!/bin/bash
# one iteration on the box: K2 + fused parity tests, the small-cloud sweep,
# the c3 headline and the per-CTA trace
set -o pipefail
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_api_r02.py -q -x 2>&1 | tail -3
SMALL_ONLY="20000 100000 400000 1600000" bash scripts/gpu_small_sweep.sh
bash scripts/gpu_small_sweep.sh 2>/dev/null | grep -E "^floor " || true
python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e --no-legs > gpurun_out/c3.json 2>/dev/null && python -c "
import json; d=json.loads(open('gpurun_out/c3.json').read().strip().splitlines()[-1]); r=d['roofline']
print('c3 step %.4f ms K %.4f frac %.3f fused %s' % (d['ms_per_step'], r['k2_ms_avg'], r['frac'], r['fused_compaction']))"
[ -n "$TRACE" ] && bash scripts/gpu_trace_k2.sh 2>&1 | grep -v "^ *[0-9] [a-z]" | head -20
exit 0
