#!/bin/bash
# per-tile phase cycles of k_assemble (GK_ASM_PROF=1), new-feature tests, F_analytic probe
mkdir -p gpurun_out
for c in "10242 P0 3 natural" "10242 P1 3 rcb" "40962 P0 3 natural"; do
  set -- $c
  p=$(GK_ORDER=$4 GK_ASM_PROF=1 timeout 150 python scripts/asm_probe.py --n $1 --fam $2 --gauss $3 --once 2>&1 | grep gk_asm_prof)
  echo "$c | $p"
done
timeout 600 python -m pytest -q -x tests/test_gpu_bigdof.py tests/test_gpu_green.py tests/test_gpu_nearfield.py > gpurun_out/pytest_ph.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ph.log
timeout 300 python scripts/fanalytic_probe.py > gpurun_out/fan_plain.log 2>&1 && \
timeout 600 ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fp64_pred_on.sum,smsp__inst_executed_pipe_xu.sum \
   -k regex:k_probe_analytic -c 1 --csv --log-file gpurun_out/r02_fanalytic_probe.csv python scripts/fanalytic_probe.py > gpurun_out/fan_ncu.log 2>&1
echo "fan rc=$?"; cat gpurun_out/fan_plain.log
