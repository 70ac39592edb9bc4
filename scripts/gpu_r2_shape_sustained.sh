#!/bin/bash
# k_assemble<.,.,16> shape (CTAs per SM, records per group) under the bench's sustained, power-capped
# step: side trees _ab/a (4, 6) and _ab/b (5, 2) against the kept (5, 3)
one() { python bench.py --extras none --no-cpu-baseline --no-e2e --steps 30 --warmup 5 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ms_per_step %.2f assembly_ms %.2f matvecs %.2f frac %.4f clk %s' % (d['ms_per_step'], d['assembly_ms'], d['matvecs_step_ms'], d['roofline']['frac'], d['clocks']['sm_mhz']))"; }
for i in 1 2; do
  echo -n "kept (5,3): "; one
  echo -n "a    (4,6): "; (cd _ab/a && one)
  echo -n "b    (5,2): "; (cd _ab/b && one)
done
