for i in 1 2; do
  echo -n "kept 2x28 xt=0: "; python scripts/mv_probe.py --n 81920 --nrhs 10 --reps 5
  echo -n "kept 2x28 xt=1: "; GK_MM_XT=1 python scripts/mv_probe.py --n 81920 --nrhs 10 --reps 5
  for v in v1 v2; do for xt in 0 1; do
    echo -n "$v xt=$xt: "; (cd _ab/$v && GK_MM_XT=$xt python scripts/mv_probe.py --n 81920 --nrhs 10 --reps 5)
  done; done
done
