#!/bin/bash
# k_assemble quick timing on cfg 4 / P1 L5 (cfg 2) / P0 L5 6-pt (cfg 3) + optional tests
r=$(timeout 300 python scripts/asm_probe.py --n 40962 --fam P0 --gauss 3 --reps 3 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('%.2f ms (%s MHz)' % (d['ms'][0], d['clocks']['sm_mhz']))")
r2=$(timeout 300 python scripts/asm_probe.py --n 10242 --fam P1 --gauss 3 --reps 5 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('%.3f' % d['ms'][0])")
r3=$(timeout 300 python scripts/asm_probe.py --n 10242 --fam P0 --gauss 6 --reps 5 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('%.3f' % d['ms'][0])")
echo "${TAG:-} cfg4 $r | P1 L5 $r2 ms | P0 L5 6pt $r3 ms"
if [ -n "$TESTS" ]; then timeout 1500 python -m pytest -q -x $TESTS 2>&1 | tail -3; fi
