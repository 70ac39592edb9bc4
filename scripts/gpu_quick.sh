#!/bin/bash
# Quick iteration on a gpurun box: one GPU test file + a short bench of one config.
# usage: bash scripts/gpu_quick.sh TAG TESTFILE CONFIG [STEPS]
TAG=$1; TF=${2:-tests/test_gpu_assembly.py}; CFG=${3:-2}; ST=${4:-10}
mkdir -p gpurun_out
timeout 900 python -m pytest $TF -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --config $CFG --steps $ST --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"; tail -2 gpurun_out/bench_$TAG.err
python - "$TAG" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/bench_{sys.argv[1]}.json"))
print({k: d.get(k) for k in ["value", "ms_per_step", "assembly_ms", "nearfield_ms", "matvec_ms", "clocks"]})
print(d.get("roofline"))
PY
