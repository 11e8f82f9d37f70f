#!/bin/bash
# ncu --set full of the step kernel for a given bench configuration.
# usage: gpu_prof.sh <tag> <kernel-regex> [bench args...]   (env passes through)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
TAG=$1; KRE=$2; shift 2
CMD="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu $@"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$KRE -s 2 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu $TAG rc=$?"
