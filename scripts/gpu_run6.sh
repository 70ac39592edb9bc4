mkdir -p gpurun_out
timeout 300 python scripts/fpair_probe.py 65536 > gpurun_out/fp6.log 2>&1 && timeout 900 ncu --set full --clock-control none -k regex:k_fast -c 1 -o gpurun_out/prof_kfast python scripts/fpair_probe.py 65536 > gpurun_out/ncu_kfast.log 2>&1; echo "ncu1 rc=$?"
CMD="python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 $CMD > gpurun_out/b6.json 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_assemble -s 3 -c 1 -o gpurun_out/prof_cfg4 $CMD > gpurun_out/ncu_cfg4.log 2>&1; echo "ncu2 rc=$?"; tail -2 gpurun_out/ncu_cfg4.log
