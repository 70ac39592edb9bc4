#!/bin/bash
# k_assemble on cfg 4: where the store time goes (GK_ASM_DBG 16: no direct stores, 32: no mirror stores, 48: neither)
for d in ${DBGS:-0 16 32 48 1}; do
  r=$(GK_ASM_DBG=$d timeout 300 python scripts/asm_probe.py --n 40962 --fam P0 --gauss 3 --reps 3 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('%.2f ms (%s MHz)' % (d['ms'][0], d['clocks']['sm_mhz']))")
  echo "dbg=$d cfg4 $r"
done
