#!/bin/bash
# multi-RHS matvec quick timing
for r in 1 2 4 5 10; do timeout 300 python scripts/mv_probe.py --n 81920 --nrhs $r --reps 3; done
timeout 300 python scripts/mv_probe.py --n 10242 --nrhs 10 --reps 10
if [ -n "$TESTS" ]; then timeout 600 python -m pytest -q -x $TESTS 2>&1 | tail -2; fi
