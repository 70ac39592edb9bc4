#!/bin/bash
# k_assemble: tiles per CTA sweep (GK_ASM_TPC) on cfg 4 / P1 L5 / P0 L5 6-pt, then the assembly tests
for tpc in 1 2 3 4; do
  GK_ASM_TPC=$tpc TAG="tpc=$tpc" bash scripts/gpu_r2_asmq.sh
done
timeout 1500 python -m pytest -q -x -m gpu tests/test_gpu_assembly.py tests/test_gpu_golden.py tests/test_gpu_stream.py 2>&1 | tail -3
