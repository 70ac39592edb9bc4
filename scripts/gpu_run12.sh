mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest12.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest12.log
timeout 900 python bench.py > gpurun_out/bench12_default.json 2> gpurun_out/bench12_default.err; echo "bench rc=$?"; cat gpurun_out/bench12_default.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench12_ref.json 2>&1; echo "ref rc=$?"; head -c 600 gpurun_out/bench12_ref.json; echo
timeout 900 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench12_cfg3.json 2>&1; echo "cfg3 rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench12_cfg3.json')); print('cfg3', d['assembly_ms'], d['nearfield_ms'], d['nearfield'], d['matvec_ms'])"
timeout 900 python bench.py --config 5 --steps 2 > gpurun_out/bench12_cfg5.json 2>&1; echo "cfg5 rc=$?"; cat gpurun_out/bench12_cfg5.json
