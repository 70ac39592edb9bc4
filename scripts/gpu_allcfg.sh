#!/bin/bash
# Bench line of every config (short runs), for DESIGN.md §5.
# usage: bash scripts/gpu_allcfg.sh TAG [CONFIGS...]
TAG=$1; shift; CFGS=${@:-1 2 3 4 5}
mkdir -p gpurun_out
for c in $CFGS; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_cfg$c.json 2> gpurun_out/bench_${TAG}_cfg$c.err
  echo "cfg$c rc=$?"
  python - "$TAG" "$c" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/bench_{sys.argv[1]}_cfg{sys.argv[2]}.json"))
keep = ["value", "unit", "ms_per_step", "assembly_ms", "nearfield_ms", "matvec_ms", "matvec_gbs", "clocks", "e2e"]
print({k: d.get(k) for k in keep})
print(d.get("roofline"))
if d.get("nearfield"): print(d["nearfield"])
PY
done
