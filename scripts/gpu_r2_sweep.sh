#!/bin/bash
# rebuild with each GK_NVCC_EXTRA variant (";"-separated in $VARIANTS) and time k_assemble
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  touch paper_1804_00995_b200/csrc/${TOUCH:-gk_assembly.cu}; GK_NVCC_EXTRA="$v" timeout 600 python paper_1804_00995_b200/build.py ${FORCE:+--force} > /tmp/build.log 2>&1 || { echo "build failed: $v"; tail -5 /tmp/build.log; continue; }
  if [ -n "$CMD" ]; then echo "[$v]"; eval "$CMD"; else TAG="[$v]" bash scripts/gpu_r2_asmq.sh; fi
done
