#!/bin/bash
# ncu --set full of k_assemble on the given mesh (default: P0 L5, the cfg-4 tile structure)
mkdir -p gpurun_out
TAG=${TAG:-x}; N=${N:-10242}; FAM=${FAM:-P0}; G=${G:-3}
timeout 300 python scripts/asm_probe.py --n $N --fam $FAM --gauss $G --once > gpurun_out/ncu_${TAG}_plain.log 2>&1 &&
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_assemble -c 1 \
  -o gpurun_out/r02_k_assemble_$TAG -f python scripts/asm_probe.py --n $N --fam $FAM --gauss $G --once > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_$TAG.log
