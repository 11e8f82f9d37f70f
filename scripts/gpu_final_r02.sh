#!/bin/bash
# Round-2 final evidence on one B200: smoke, full GPU tests, the bench as the
# driver runs it (plain, torchrun N=1 through ShardedAdamWGS, reference arm),
# the launch list, the drop-in timing.
mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; tail -1 gpurun_out/final/smoke.log
python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/final/pytest_gpu.log; cat gpurun_out/final/pytest_gpu.log
python bench.py --steps 20 --warmup 5 > gpurun_out/final/bench_c3.json 2> gpurun_out/final/bench_c3.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu > gpurun_out/final/bench_c3_torchrun_n1.json 2> gpurun_out/final/bench_c3_torchrun_n1.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 1 --steps 20 --warmup 5 --sharded --no-cpu --no-e2e > gpurun_out/final/bench_c3_sharded_n1.json 2> gpurun_out/final/bench_c3_sharded_n1.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final/bench_c3_reference.json 2> gpurun_out/final/bench_c3_reference.err
python scripts/adopt_bench.py > gpurun_out/final/adopt_dropin_c3.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches_c3.csv python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-legs > /dev/null 2>&1
python - <<'PY'
import json
for f in ["bench_c3", "bench_c3_torchrun_n1", "bench_c3_sharded_n1", "bench_c3_reference"]:
    try:
        d = json.loads(open(f"gpurun_out/final/{f}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "FAILED", e); continue
    r = d.get("roofline") or {}
    e2e = (d.get("e2e") or {}).get("value")
    print(f, "value %.4g ms %.4f frac %s e2e %s launches %s clocks %s" % (d["value"], d["ms_per_step"], r.get("frac"), e2e, d.get("gpu_launches"), d.get("clocks")))
PY
cat gpurun_out/final/adopt_dropin_c3.txt
