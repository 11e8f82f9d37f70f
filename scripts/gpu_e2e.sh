#!/bin/bash
# Pinned-host gradient tests + default bench (with e2e) on one B200.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_reference_api.py -m gpu -x -q -k "pinned" > gpurun_out/pytest_pinned.log 2>&1; echo "pinned rc=$?"; tail -3 gpurun_out/pytest_pinned.log
timeout 600 python bench.py $BENCH_ARGS > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; echo "bench rc=$?"
tail -c 2500 gpurun_out/bench_e2e.json; tail -5 gpurun_out/bench_e2e.err
