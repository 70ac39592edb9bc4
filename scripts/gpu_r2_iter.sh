#!/bin/bash
# round 2 iteration: assembly parity tests + k_assemble timings on P0 L5 / cfg 4 / P1 L5
mkdir -p gpurun_out
TAG=${1:-it}
timeout 900 python -m pytest -x -q tests/test_gpu_assembly.py tests/test_gpu_stream.py tests/test_gpu_golden.py > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
for c in "10242 P0 3" "40962 P0 3" "10242 P1 3" "10242 P0 6"; do
for env in ${ENVS:-"GK_X=0"}; do
  set -- $c
  r=$(env ${env//,/ } timeout 300 python scripts/asm_probe.py --n $1 --fam $2 --gauss $3 --reps 5 2>&1 | tail -1)
  echo "$c $env $(echo $r | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('ms %.3f eval/u %.3f tiles %d mhz %s' % (d['ms'][0], d['pairs_evaluated']/d['pairs_unique'], d['tiles'], d['clocks']['sm_mhz']))" 2>&1)"
done; done
