bash scripts/gpu_ncu_full.sh r32nf 3 k_nearfield 0
bash scripts/gpu_ncu_full.sh r32g 5 k_green64 0
