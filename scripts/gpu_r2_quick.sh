#!/bin/bash
# quick: phase profile + timings of k_assemble (P0 L5, cfg 4, P1 L5, P0 L5 6-pt) and the assembly tests
mkdir -p gpurun_out
for c in "10242 P0 3" "40962 P0 3" "10242 P1 3" "10242 P0 6"; do
  set -- $c
  p=$(GK_ASM_PROF=1 timeout 150 python scripts/asm_probe.py --n $1 --fam $2 --gauss $3 --once 2>&1 | grep gk_asm_prof)
  r=$(timeout 200 python scripts/asm_probe.py --n $1 --fam $2 --gauss $3 --reps 5 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('ms %.3f eval/u %.3f tiles %d' % (d['ms'][0], d['pairs_evaluated']/d['pairs_unique'], d['tiles']))")
  echo "$c | $r | $p"
done
if [ -n "$TESTS" ]; then timeout 900 python -m pytest -q -x $TESTS > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_q.log; fi
