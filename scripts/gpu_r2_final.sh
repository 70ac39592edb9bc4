#!/bin/bash
# round-2 evidence of the final kernels: full-size parity log, ncu --set full of
# k_assemble (P0 L5 = the cfg-4 tile structure), cfg-4 application-replay
# metrics of k_assemble, matvec_multi dram bytes, the launch list of a short
# cfg-4 bench.
mkdir -p gpurun_out
TAG=${TAG:-f}
if [ -z "$NOPARITY" ]; then rm -f gpurun_out/parity_$TAG.jsonl
GK_PARITY_LOG=gpurun_out/parity_$TAG.jsonl timeout 2400 python -m pytest -q -x -s tests/test_gpu_full_parity.py > gpurun_out/pytest_parity_$TAG.log 2>&1
echo "parity rc=$?"; tail -2 gpurun_out/pytest_parity_$TAG.log; fi
timeout 300 python scripts/asm_probe.py --n 10242 --fam P0 --once > /dev/null 2>&1 &&
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_assemble -c 1 \
  -o gpurun_out/r02_k_assemble_p0l5_$TAG -f python scripts/asm_probe.py --n 10242 --fam P0 --once > gpurun_out/ncu_p0l5_$TAG.log 2>&1
echo "ncu p0l5 rc=$?"
timeout 1800 ncu --replay-mode application --clock-control none -k regex:k_assemble -c 1 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second \
  --csv --log-file gpurun_out/r02_k_assemble_cfg4_metrics_$TAG.csv python scripts/asm_probe.py --n 40962 --fam P0 --once > gpurun_out/ncu4_$TAG.log 2>&1
echo "ncu cfg4 rc=$?"
timeout 900 ncu --clock-control none -k regex:k_matvec_multi -c 2 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
  --csv --log-file gpurun_out/r02_matvec_multi_cfg4_$TAG.csv python scripts/mv_probe.py --n 81920 --nrhs 10 --reps 0 > /dev/null 2>&1
echo "ncu mm rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_cfg4_$TAG.csv \
  python bench.py --extras none --no-cpu-baseline --no-e2e --steps 2 --warmup 3 > gpurun_out/ncu_bench_$TAG.log 2>&1
echo "launch list rc=$?"
