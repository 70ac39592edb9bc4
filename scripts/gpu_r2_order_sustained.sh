#!/bin/bash
# dof order (natural / RCB units of 4 / RCB) for cfg 4 under the bench's sustained, power-capped step
one() { python bench.py --extras none --no-cpu-baseline --no-e2e --steps 30 --warmup 5 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ms_per_step %.2f assembly_ms %.2f matvecs %.2f frac %.4f clk %s halo %.3f' % (d['ms_per_step'], d['assembly_ms'], d['matvecs_step_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['pairs_evaluated_per_unique']))"; }
for i in 1 2; do
  echo -n "natural: "; one
  echo -n "rcb4   : "; GK_ORDER=rcb4 one
  echo -n "rcb    : "; GK_ORDER=rcb one
done
