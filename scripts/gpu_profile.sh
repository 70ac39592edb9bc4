#!/bin/bash
# ncu evidence for the bench command (run only after it exits 0 plainly):
#  1. the launch list (gpu__time_duration per launch, clocks uncontrolled),
#  2. one --set full capture of the top kernel (K1+K2 k_assemble).
# usage: bash scripts/gpu_profile.sh TAG [CONFIG] [KERNEL_REGEX]
TAG=${1:-x}; CFG=${2:-2}; KRE=${3:-k_assemble}
mkdir -p gpurun_out
ARGS="--config $CFG --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 python bench.py $ARGS > gpurun_out/plain_$TAG.json 2>&1; rc=$?; echo "plain rc=$rc"
[ $rc -eq 0 ] || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py $ARGS > gpurun_out/ncu_list_$TAG.log 2>&1
echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$KRE -s ${SKIP:-0} -c 1 \
  -o gpurun_out/full_$TAG -f python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full rc=$?"; tail -3 gpurun_out/ncu_full_$TAG.log
