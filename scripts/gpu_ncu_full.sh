#!/bin/bash
# One ncu --set full capture of a kernel in the bench command.
# usage: bash scripts/gpu_ncu_full.sh TAG CONFIG KERNEL_REGEX SKIP
TAG=$1; CFG=${2:-2}; KRE=${3:-k_assemble}; SKIP=${4:-0}
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$KRE -s $SKIP -c 1 \
  -o gpurun_out/full_$TAG -f python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full rc=$?"; tail -2 gpurun_out/ncu_full_$TAG.log
