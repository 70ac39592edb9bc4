#!/bin/bash
mkdir -p gpurun_out
bash scripts/gpu_r2_iter.sh b1
( time timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_b1.json 2> gpurun_out/bench_b1.err ) 2> gpurun_out/bench_b1.time
echo "bench rc=$?"; tail -3 gpurun_out/bench_b1.err; cat gpurun_out/bench_b1.time
timeout 300 python scripts/asm_probe.py --n 10242 --fam P0 --once > gpurun_out/b1_once.log 2>&1 &&
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_assemble -c 1 \
  -o gpurun_out/r02_k_assemble_p0l5_b1 -f python scripts/asm_probe.py --n 10242 --fam P0 --once > gpurun_out/b1_ncu.log 2>&1
echo "ncu rc=$?"
