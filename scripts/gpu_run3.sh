mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_assembly.py -q -x > gpurun_out/pytest3.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest3.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/bench3.json 2>&1; echo "plain rc=$?"; cat gpurun_out/bench3.json
for c in 1 3 4; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench3_cfg$c.json 2>&1; echo "cfg$c rc=$?"; cat gpurun_out/bench3_cfg$c.json | head -c 1500; echo; done
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_assemble -s 2 -c 1 -o gpurun_out/prof_asm_r01b $CMD > gpurun_out/ncu_full3.log 2>&1; echo "ncu rc=$?"
