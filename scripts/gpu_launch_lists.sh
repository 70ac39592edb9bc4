mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv \
  python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_cfg4.log 2>&1
echo "rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv \
  python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_cfg3.log 2>&1
echo "rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv \
  python bench.py --config 5 --steps 1 --warmup 3 > gpurun_out/ncu_cfg5.log 2>&1
echo "rc=$?"
