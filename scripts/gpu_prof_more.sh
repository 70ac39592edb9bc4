#!/bin/bash
# ncu --set full captures of the K3 (cfg 3) and K5 (cfg 5) kernels for profiles/.
bash scripts/gpu_ncu_full.sh r49nf 3 k_nearfield 0
bash scripts/gpu_ncu_full.sh r49g 5 k_green64_sym 2
