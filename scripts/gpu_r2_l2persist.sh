#!/bin/bash
# k_assemble with the plan tables in a persisting L2 window (default) vs GK_L2_PERSIST=0; cfg 4 / P1 L5 / P0 L5 6-pt,
# then the cfg-2 (P1 L5) DRAM bytes both ways
for i in 1 2; do
  GK_L2_PERSIST=0 TAG="plain  " bash scripts/gpu_r2_asmq.sh
  TAG="persist" bash scripts/gpu_r2_asmq.sh
done
for p in 0 1; do
GK_L2_PERSIST=$p timeout 900 ncu --clock-control none -k regex:k_assemble -c 1 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --csv --log-file gpurun_out/s5_l2persist_cfg2_$p.csv python scripts/asm_probe.py --n 10242 --fam P1 --once > /dev/null 2>&1
echo "cfg2 GK_L2_PERSIST=$p"; grep '^"' gpurun_out/s5_l2persist_cfg2_$p.csv | awk -F'","' '{print $13, $15}'
done
python -m pytest -q -x tests/test_gpu_assembly.py tests/test_gpu_stream.py tests/test_gpu_bigdof.py tests/test_gpu_golden.py tests/test_gpu_shard.py 2>&1 | tail -2
