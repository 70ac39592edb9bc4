#!/bin/bash
# timing experiments (GK_ASM_DBG bits: 1 no stores, 2 no gather, 4 general gather path)
for n in ${NS:-10242 40962}; do for d in ${DBGS:-0 4}; do
  p=$(GK_ASM_DBG=$d GK_ASM_PROF=1 timeout 150 python scripts/asm_probe.py --n $n --fam P0 --gauss 3 --once 2>&1 | grep gk_asm_prof)
  r=$(GK_ASM_DBG=$d timeout 200 python scripts/asm_probe.py --n $n --fam P0 --gauss 3 --reps 5 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('ms %.3f' % d['ms'][0])")
  echo "$n dbg=$d | $r | $p"
done; done
