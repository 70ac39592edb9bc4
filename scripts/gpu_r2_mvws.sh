#!/bin/bash
# multi-RHS matvec: warp-specialised kernel (GK_MM_WS=1) stage-shape sweep against the kept kernel, 10 vectors on cfg 4
GK_MM_WS=1 timeout 600 python -m pytest -q -x tests/test_gpu_assembly.py -k "matvec" 2>&1 | tail -2
for i in 1 2; do
  echo -n "kept: "; timeout 300 python scripts/mv_probe.py --n 81920 --nrhs 10 --reps 5
  for cfg in ${SHAPES:-"4 4" "7 2" "5 3" "3 5" "2 8" "8 2"}; do
    set -- $cfg
    echo -n "ws cols=$1 nst=$2: "; GK_MM_WS=1 GK_MM_COLS=$1 GK_MM_NST=$2 timeout 300 python scripts/mv_probe.py --n 81920 --nrhs 10 --reps 5
  done
done
