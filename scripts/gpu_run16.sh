mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nearfield.py -q -x > gpurun_out/pytest16.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest16.log
timeout 300 python scripts/nf_probe.py > gpurun_out/nf16.log 2>&1; cat gpurun_out/nf16.log
