#!/bin/bash
# k_assemble with the plan tables in a persisting L2 window (GK_L2_PERSIST=1) vs without; cfg 4 / P1 L5 / P0 L5 6-pt
for i in 1 2; do
  TAG="plain  " bash scripts/gpu_r2_asmq.sh
  GK_L2_PERSIST=1 TAG="persist" bash scripts/gpu_r2_asmq.sh
done
GK_L2_PERSIST=1 timeout 900 ncu --replay-mode application --clock-control none -k regex:k_assemble -c 1 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --csv --log-file gpurun_out/s5_l2persist_cfg4.csv python scripts/asm_probe.py --n 40962 --fam P0 --once > /dev/null 2>&1
grep '^"' gpurun_out/s5_l2persist_cfg4.csv | awk -F'","' '{print $13, $15}'
