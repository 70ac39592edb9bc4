#!/bin/bash
# k_assemble timing experiments on cfg 4 (GK_ASM_DBG: 1 no stores, 2 no gather, 4 no pair loop, 8 no RMW)
for d in 0 1 2 4 8 12 6; do
  r=$(GK_ASM_DBG=$d timeout 300 python scripts/asm_probe.py --n ${N:-40962} --fam P0 --gauss 3 --reps 3 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('ms %.2f  clk %s' % (d['ms'][0], d['clocks']['sm_mhz']))")
  echo "dbg=$d $r"
done
