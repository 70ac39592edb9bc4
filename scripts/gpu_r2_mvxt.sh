#!/bin/bash
# multi-RHS matvec: X transposed beforehand so a stage's x values come in one bulk copy (GK_MM_XT=1) vs ten
GK_MM_XT=1 timeout 600 python -m pytest -q -x tests/test_gpu_assembly.py -k "matvec" 2>&1 | tail -2
for i in 1 2; do
  for r in 10 6 3; do
    echo -n "kept nrhs=$r: "; timeout 300 python scripts/mv_probe.py --n 81920 --nrhs $r --reps 5
    echo -n "xt   nrhs=$r: "; GK_MM_XT=1 timeout 300 python scripts/mv_probe.py --n 81920 --nrhs $r --reps 5
  done
done
