#!/bin/bash
# round 2: k_assemble time vs tile layout knobs (P0 L5 = cfg-4 tile structure, and cfg 4)
mkdir -p gpurun_out
for n in 10242 40962; do
for env in "GK_X=0" "GK_ORDER=rcb GK_XCUT=1" "GK_ORDER=rcb GK_XCUT=1 GK_UNIT=4" "GK_ORDER=rcb GK_XCUT=1 GK_UNIT=2" "GK_ORDER=natural GK_XCUT=1"; do
  echo "== $n $env" >> gpurun_out/lay.log
  env $env timeout 300 python scripts/asm_probe.py --n $n --fam P0 --reps 5 >> gpurun_out/lay.log 2>&1
done; done
for env in "GK_X=0" "GK_ORDER=rcb GK_XCUT=1"; do
  echo "== P1 $env" >> gpurun_out/lay.log
  env $env timeout 300 python scripts/asm_probe.py --n 10242 --fam P1 --reps 5 >> gpurun_out/lay.log 2>&1
done
cat gpurun_out/lay.log | python -c "
import sys,json
for l in sys.stdin:
  if l.startswith('=='): print(l.strip(), end=' ')
  elif l.startswith('{'):
    d=json.loads(l); print('ms %.3f eval/u %.3f tiles %d mhz %s' % (d['ms'][0], d['pairs_evaluated']/d['pairs_unique'], d['tiles'], d['clocks']['sm_mhz']))
"
