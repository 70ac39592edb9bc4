#!/bin/bash
# round 2, probe 1: k_assemble per-evaluated-pair rate on P1 L5 / P0 L5 / P0 L6 (cfg 4),
# then ncu --set full of the P0 L5 3-pt kernel (same tile structure as cfg 4)
# and a two-metric application-replay capture of cfg 4 itself.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
for c in "--n 10242 --fam P1" "--n 10242 --fam P0" "--n 40962 --fam P0"; do
  timeout 300 python scripts/asm_probe.py $c --reps 5 >> gpurun_out/p1_rates.jsonl 2>>gpurun_out/p1_rates.err; echo "rc=$? $c"
done
cat gpurun_out/p1_rates.jsonl
timeout 300 python scripts/asm_probe.py --n 10242 --fam P0 --once > gpurun_out/p1_once.log 2>&1 &&
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_assemble -c 1 \
  -o gpurun_out/r02_k_assemble_p0l5 -f python scripts/asm_probe.py --n 10242 --fam P0 --once > gpurun_out/p1_ncu.log 2>&1
echo "ncu1 rc=$?"; tail -3 gpurun_out/p1_ncu.log
timeout 300 python scripts/asm_probe.py --n 40962 --fam P0 --once > gpurun_out/p1_once4.log 2>&1 &&
timeout 1500 ncu --replay-mode application --clock-control none -k regex:k_assemble -c 1 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum,sm__warps_active.avg.pct_of_peak_sustained_active \
  --csv --log-file gpurun_out/r02_k_assemble_cfg4_metrics.csv python scripts/asm_probe.py --n 40962 --fam P0 --once > gpurun_out/p1_ncu4.log 2>&1
echo "ncu4 rc=$?"; tail -3 gpurun_out/p1_ncu4.log
