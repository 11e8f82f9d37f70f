#!/bin/bash
# Round-end evidence on one B200: smoke + GPU tests, the bench lines
# (c3 headline with e2e and the CPU port, coherent / per-attribute c3, c1,
# c2, c4), the ncu launch list and one --set full capture of K2, the c5
# visibility sweep, the reference arm and a torchrun N=1 line.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
bash scripts/gpu_tests.sh
bash scripts/gpu_bench.sh
bash scripts/gpu_c5_sweep.sh
python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo "ref rc=$?"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 1 --no-cpu > gpurun_out/final_tr.json 2> gpurun_out/final_tr.err; echo "torchrun rc=$?"
