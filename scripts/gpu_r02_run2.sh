#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -8 > gpurun_out/pytest_gpu_full.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 20 --warmup 5 --sharded --no-cpu > gpurun_out/bench_c3_sharded_n1.json 2> gpurun_out/bench_c3_sharded_n1.err
cat gpurun_out/pytest_gpu_full.log
tail -c 300 gpurun_out/bench_c3_sharded_n1.json; grep -v "NCCL INFO" gpurun_out/bench_c3_sharded_n1.err | tail -5
bash scripts/gpu_evidence.sh
