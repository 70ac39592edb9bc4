mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/b9.json 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_assemble -s 2 -c 1 -o gpurun_out/prof_asm_r01c $CMD > gpurun_out/ncu9.log 2>&1; echo "ncu rc=$?"
