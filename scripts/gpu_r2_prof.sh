#!/bin/bash
# round-2 evidence pass: k_assemble phase cycles on cfg 4, ncu --set full of the
# P0 L5 k_assemble (cfg-4 tile structure), cfg-4 application-replay metrics of
# k_assemble, dram bytes of the stored matvec (cfg 2, cfg 4), the F_analytic
# probe, compute-sanitizer (memcheck, racecheck, synccheck) on small meshes, and
# the launch list of a short cfg-4 bench.
mkdir -p gpurun_out
TAG=${TAG:-p}
free -g > gpurun_out/host_$TAG.txt; nproc >> gpurun_out/host_$TAG.txt; lscpu | grep -i "model name" >> gpurun_out/host_$TAG.txt
GK_ASM_PROF=1 timeout 300 python scripts/asm_probe.py --n 40962 --fam P0 --gauss 3 --once 2>&1 | grep gk_asm_prof > gpurun_out/phase_cfg4_$TAG.txt
echo "phase rc=$?"; cat gpurun_out/phase_cfg4_$TAG.txt
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python scripts/sanitize_probe.py > gpurun_out/sanitizer_${t}_$TAG.log 2>&1
  echo "sanitizer $t rc=$?"; tail -4 gpurun_out/sanitizer_${t}_$TAG.log
done
timeout 300 python scripts/mv_probe.py --n 10242 --reps 5 && timeout 300 python scripts/mv_probe.py --n 81920 --reps 3
timeout 600 ncu --clock-control none -k regex:k_matvec -c 4 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
  --csv --log-file gpurun_out/r02_matvec_cfg2_$TAG.csv python scripts/mv_probe.py --n 10242 --reps 1 > /dev/null 2>&1
echo "ncu mv2 rc=$?"
timeout 900 ncu --clock-control none -k regex:k_matvec -c 2 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --csv --log-file gpurun_out/r02_matvec_cfg4_$TAG.csv python scripts/mv_probe.py --n 81920 --reps 0 > /dev/null 2>&1
echo "ncu mv4 rc=$?"
timeout 300 python scripts/asm_probe.py --n 10242 --fam P0 --once > /dev/null 2>&1 &&
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_assemble -c 1 \
  -o gpurun_out/r02_k_assemble_p0l5_$TAG -f python scripts/asm_probe.py --n 10242 --fam P0 --once > gpurun_out/ncu_p0l5_$TAG.log 2>&1
echo "ncu p0l5 rc=$?"; tail -2 gpurun_out/ncu_p0l5_$TAG.log
timeout 1800 ncu --replay-mode application --clock-control none -k regex:k_assemble -c 1 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second \
  --csv --log-file gpurun_out/r02_k_assemble_cfg4_metrics_$TAG.csv python scripts/asm_probe.py --n 40962 --fam P0 --once > gpurun_out/ncu4_$TAG.log 2>&1
echo "ncu cfg4 rc=$?"; tail -2 gpurun_out/ncu4_$TAG.log
timeout 300 python scripts/fanalytic_probe.py > gpurun_out/fan_plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fp64_pred_on.sum,smsp__inst_executed_pipe_xu.sum \
   -k regex:k_probe_analytic -c 1 --csv --log-file gpurun_out/r02_fanalytic_probe_$TAG.csv python scripts/fanalytic_probe.py > gpurun_out/fan_ncu_$TAG.log 2>&1
echo "fan rc=$?"; cat gpurun_out/fan_plain_$TAG.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_cfg4_$TAG.csv \
  python bench.py --extras none --no-cpu-baseline --no-e2e --steps 2 --warmup 3 > gpurun_out/ncu_bench_$TAG.log 2>&1
echo "launch list rc=$?"
