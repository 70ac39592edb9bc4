mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_assembly.py -q -x > gpurun_out/pytest10.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest10.log
for c in 2 3 4; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench10_cfg$c.json 2>&1; echo "cfg$c rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench10_cfg$c.json')); print('cfg$c', 'asm_ms', round(d['assembly_ms'],3), 'mv_ms', round(d['matvec_ms'],3), 'frac', round(d['roofline']['frac'],3), 'halo', round(d['pairs_evaluated_per_unique'],3), 'clk', d['clocks'])"; done
