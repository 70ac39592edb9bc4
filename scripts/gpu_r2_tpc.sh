#!/bin/bash
# k_assemble: tiles per CTA (GK_ASM_TPC) against the HEAD build under _ab/base, then the assembly tests
python -m pytest -q -x tests/test_gpu_assembly.py tests/test_gpu_stream.py tests/test_gpu_bigdof.py tests/test_gpu_golden.py 2>&1 | tail -3
for i in ${PASSES:-1}; do
  (cd _ab/base && TAG="base" bash scripts/gpu_r2_asmq.sh)
  for tpc in ${TPCS:-1 2 4 8}; do GK_ASM_TPC=$tpc TAG="new tpc=$tpc" bash scripts/gpu_r2_asmq.sh; done
done
