#!/bin/bash
# Round-2 check on one B200: the new GPU tests, then the bench (plain, the
# ShardedAdamWGS path on one rank under torchrun).
mkdir -p gpurun_out
python -m pytest tests/test_gpu_api_r02.py tests/test_gpu_sharded.py tests/test_gpu_multistep.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -30 > gpurun_out/pytest_r02.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 20 --warmup 5 --sharded --no-cpu > gpurun_out/bench_c3_sharded_n1.json 2> gpurun_out/bench_c3_sharded_n1.err
tail -5 gpurun_out/pytest_r02.log
tail -c 600 gpurun_out/bench_c3.json; tail -3 gpurun_out/bench_c3.err
tail -c 400 gpurun_out/bench_c3_sharded_n1.json; tail -5 gpurun_out/bench_c3_sharded_n1.err
