#!/bin/bash
# A/B on one box: the HEAD build under _ab/base (git worktree, git-ignored) against the working tree
for i in 1 2; do
  (cd _ab/base && TAG="base" bash scripts/gpu_r2_asmq.sh)
  for tpc in ${TPCS:-1 3}; do GK_ASM_TPC=$tpc TAG="new tpc=$tpc" bash scripts/gpu_r2_asmq.sh; done
done
