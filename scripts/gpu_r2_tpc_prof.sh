(cd _ab/base && GK_ASM_PROF=1 python scripts/asm_probe.py --n 40962 --fam P0 --gauss 3 --once 2>&1 | grep gk_asm_prof)
for tpc in 1 2 4; do GK_ASM_TPC=$tpc GK_ASM_PROF=1 python scripts/asm_probe.py --n 40962 --fam P0 --gauss 3 --once 2>&1 | grep gk_asm_prof; done
