#!/bin/bash
# multi-RHS matvec: tests, probe timings, short cfg-4 bench
mkdir -p gpurun_out
TAG=${TAG:-mv}
timeout 600 python -m pytest -q -x tests/test_gpu_assembly.py -k matvec > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log
for r in 1 2 4 10; do timeout 300 python scripts/mv_probe.py --n 81920 --nrhs $r --reps 3; done
timeout 900 python bench.py --extras none --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_$TAG.err
python - <<'PY'
import json,sys
d=json.load(open("gpurun_out/bench_%s.json" % sys.argv[1] if len(sys.argv)>1 else "gpurun_out/bench_mv.json"))
print({k:d.get(k) for k in ("value","ms_per_step","assembly_ms","matvec_ms","matvecs_step_ms")})
print(d.get("roofline_matvec_multi")); print(d["roofline"]["frac"], d["clocks"]); print(d.get("e2e"))
PY
