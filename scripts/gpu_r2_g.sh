#!/bin/bash
# k_assemble gather-unit width sweep (GK_GATHER_G) on cfg 4 and P1 L5, plus parity spot check
for G in ${GS:-2 4 6 8 12 22}; do
  r=$(GK_GATHER_G=$G timeout 300 python scripts/asm_probe.py --n 40962 --fam P0 --gauss 3 --reps 3 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('%.2f' % d['ms'][0])")
  r2=$(GK_GATHER_G=$G timeout 300 python scripts/asm_probe.py --n 10242 --fam P1 --gauss 3 --reps 5 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('%.3f' % d['ms'][0])")
  r3=$(GK_GATHER_G=$G timeout 300 python scripts/asm_probe.py --n 10242 --fam P0 --gauss 6 --reps 5 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('%.3f' % d['ms'][0])")
  echo "G=$G cfg4 $r ms | P1 L5 $r2 ms | P0 L5 6pt $r3 ms"
done
if [ -n "$TESTS" ]; then timeout 900 python -m pytest -q -x $TESTS 2>&1 | tail -2; fi
