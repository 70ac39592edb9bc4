#!/bin/bash
# default bench (cfg 4 headline + cfg 2/3/5 lines) and the reference arm, as the driver runs them
mkdir -p gpurun_out
TAG=${TAG:-b}
( time timeout 1500 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err ) 2> gpurun_out/bench_$TAG.time
echo "bench rc=$?"; tail -2 gpurun_out/bench_$TAG.err; grep real gpurun_out/bench_$TAG.time
if [ -z "$NOREF" ]; then
( time timeout 1500 python bench.py --impl reference > gpurun_out/ref_$TAG.json 2> gpurun_out/ref_$TAG.err ) 2> gpurun_out/ref_$TAG.time
echo "ref rc=$?"; tail -2 gpurun_out/ref_$TAG.err; grep real gpurun_out/ref_$TAG.time
fi
