mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest17.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest17.log
timeout 900 python bench.py > gpurun_out/bench17.json 2> gpurun_out/bench17.err; echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench17.json')); print({k: d[k] for k in ['value','ms_per_step','assembly_ms','matvec_ms','clocks','e2e','cpu_baseline','gpu_launches']}); print(d['roofline'])"
