"""Time k_assemble alone on one mesh/space (CUDA events, clocks sampled).

  python scripts/asm_probe.py --n 40962 --fam P0 --gauss 3 [--reps 5] [--once]

--once: one assemble and exit (for ncu captures: -k regex:k_assemble -c 1).
Prints one JSON line per case: ms, evaluated/unique pairs, rate per evaluated
pair at the sampled clock.
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1804_00995_b200 as g  # noqa: E402
from bench import ClockSampler  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=40962)
p.add_argument("--fam", default="P0")
p.add_argument("--gauss", type=int, default=3)
p.add_argument("--laplace", action="store_true")
p.add_argument("--reps", type=int, default=5)
p.add_argument("--once", action="store_true")
a = p.parse_args()

mesh = g.build_sphere(a.n, 1.0)
hbar = g.edge_stats(mesh).mean_len
k = 0.0 if a.laplace else 2 * math.pi / (10 * hbar)
kern = g.green_kernel("[1/r]" if a.laplace else "[exp(ikr)/r]", k)
dom = g.make_domain(mesh, a.gauss)
sp = g.make_fem(mesh, a.fam)
o = g.BemOptions()
o.memory_cap_bytes = 10 ** 15
plan = g.AssemblyPlan(dom, dom, sp, kern, sp, o)
info = plan.info()
n = info["rows"]
A = torch.empty(n * n, dtype=torch.complex128, device="cuda")
s = torch.cuda.current_stream()
if a.once:
    plan.assemble(A.data_ptr(), n, s.cuda_stream)
    torch.cuda.synchronize()
    sys.exit(0)
for _ in range(2):
    plan.assemble(A.data_ptr(), n, s.cuda_stream)
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.reps)]
with ClockSampler(0) as clk:
    for e0, e1 in ev:
        e0.record(s)
        plan.assemble(A.data_ptr(), n, s.cuda_stream)
        e1.record(s)
    torch.cuda.synchronize()
ms = sorted(e0.elapsed_time(e1) for e0, e1 in ev)
c = clk.summary()
mhz = c["sm_mhz"] or 1965.0
print(json.dumps({"n": a.n, "fam": a.fam, "gauss": a.gauss, "ms": ms, "tiles": info["tiles"],
                  "pairs_evaluated": info["pairs_evaluated"], "pairs_unique": info["pairs_unique"],
                  "eval_per_s": info["pairs_evaluated"] / (ms[0] * 1e-3),
                  "eval_per_s_at_1965": info["pairs_evaluated"] / (ms[0] * 1e-3) * 1965.0 / mhz,
                  "clocks": c}))
