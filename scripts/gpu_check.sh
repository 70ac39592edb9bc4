#!/bin/bash
# Round check on a gpurun box: GPU parity suite + default bench line.
# usage: bash scripts/gpu_check.sh TAG [pytest-args...]
TAG=${1:-x}; shift
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q "$@" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python - "$TAG" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/bench_{sys.argv[1]}.json"))
print({k: d.get(k) for k in ["value", "ms_per_step", "assembly_ms", "matvec_ms", "clocks", "e2e", "gpu_launches"]})
print(d.get("roofline"))
PY
