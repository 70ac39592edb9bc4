mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests/test_gpu_nearfield.py -q -x > gpurun_out/pytest2.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest2.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/bench2_plain.json 2>&1; echo "plain rc=$?"; cat gpurun_out/bench2_plain.json
timeout 300 python scripts/fpair_probe.py 4096 > gpurun_out/fpair_plain.log 2>&1; echo "fpair rc=$?"; cat gpurun_out/fpair_plain.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_r01.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_assemble -s 2 -c 1 -o gpurun_out/prof_asm_r01 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
timeout 600 ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,gpu__time_duration.sum --csv --log-file gpurun_out/fpair_ncu.csv python scripts/fpair_probe.py 4096 > gpurun_out/fpair_ncu.log 2>&1; echo "ncu3 rc=$?"
tail -3 gpurun_out/ncu_full.log
