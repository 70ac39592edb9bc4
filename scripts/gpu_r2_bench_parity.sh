#!/bin/bash
# full default bench (cfg 4 headline + cfg 2/3/5 lines) then the full-size parity suite
mkdir -p gpurun_out
TAG=${TAG:-bp}
( time timeout 1500 python bench.py --steps ${STEPS:-10} --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err ) 2> gpurun_out/bench_$TAG.time
echo "bench rc=$?"; tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.time | grep real
if [ -z "$NOPARITY" ]; then
  rm -f gpurun_out/parity_$TAG.jsonl
  GK_PARITY_LOG=gpurun_out/parity_$TAG.jsonl timeout 2400 python -m pytest -q -x -s tests/test_gpu_full_parity.py > gpurun_out/pytest_parity_$TAG.log 2>&1
  echo "parity rc=$?"; tail -3 gpurun_out/pytest_parity_$TAG.log; cat gpurun_out/parity_$TAG.jsonl
fi
