#!/bin/bash
# round-2 checkpoint: the whole -m gpu suite, then the default bench (cfg 4 headline + extras)
mkdir -p gpurun_out
TAG=${TAG:-all}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/smi_$TAG.txt 2>&1
( time timeout 2400 python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/pytest_gpu_$TAG.log 2>&1 ) 2> gpurun_out/pytest_gpu_$TAG.time
echo "pytest rc=$?"; tail -30 gpurun_out/pytest_gpu_$TAG.log | grep -v "^$" | tail -32
if [ -z "$NOBENCH" ]; then
( time timeout 1500 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err ) 2> gpurun_out/bench_$TAG.time
echo "bench rc=$?"; tail -3 gpurun_out/bench_$TAG.err; grep real gpurun_out/bench_$TAG.time
fi
