mkdir -p gpurun_out
timeout 300 python scripts/nf_probe.py > gpurun_out/nf_plain.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_nearfield -s 1 -c 1 -o gpurun_out/prof_nf python scripts/nf_probe.py > gpurun_out/ncu_nf.log 2>&1; echo "ncu rc=$?"; cat gpurun_out/nf_plain.log
