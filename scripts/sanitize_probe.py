"""Small invocations of every device kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck) on the GPU box:

  compute-sanitizer --tool memcheck python scripts/sanitize_probe.py

k_assemble (P0 and P1, Helmholtz and Laplace, masked and unmasked tiles,
symmetric and non-symmetric plans, the 6-point rule on a perturbed mesh),
k_nearfield_b + k_nf_reduce/k_nf_apply (P0, P1), k_nf_points,
k_green64/32 and the symmetric k_green64_sym/k_green32_sym, k_matvec,
k_block_eval.  Prints one line per case."""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_00995_b200 as g  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.current_stream().cuda_stream
mesh = g.build_sphere(162, 1.0)
pmesh = g.perturb_radial(mesh, 2, 0.02)
hbar = g.edge_stats(mesh).mean_len
k = 2 * math.pi / (10 * hbar)


def assemble(m, gauss, fam, name, kk, other=None):
    d = g.make_domain(m, gauss)
    sp = g.make_fem(m, fam)
    dy, spy = (d, sp) if other is None else other
    plan = g.AssemblyPlan(d, dy, sp, g.green_kernel(name, kk), spy)
    inf = plan.info()
    r, c = inf["rows"], inf["cols"]
    A = torch.empty(r * c, dtype=torch.complex128, device="cuda")
    plan.assemble(A.data_ptr(), r, s)
    x = torch.ones(c, dtype=torch.complex128, device="cuda")
    y = torch.empty(r, dtype=torch.complex128, device="cuda")
    g.matvec(A.data_ptr(), r, c, r, x.data_ptr(), y.data_ptr(), s)
    torch.cuda.synchronize()
    print(f"assemble {fam} g{gauss} {name}: {r}x{c} tiles={inf['tiles']} |y|={float(y.abs().sum()):.6e}")


assemble(mesh, 3, "P0", "[exp(ikr)/r]", k)
assemble(mesh, 3, "P1", "[exp(ikr)/r]", k)
assemble(mesh, 3, "P1", "[1/r]", 0.0)
assemble(pmesh, 6, "P0", "[exp(ikr)/r]", k)
assemble(mesh, 7, "P1", "[exp(ikr)/r]", k, other=(g.make_domain(pmesh, 3), g.make_fem(pmesh, "P0")))

for fam, gauss in (("P0", 6), ("P1", 3)):
    d = g.make_domain(pmesh, gauss)
    sp = g.make_fem(pmesh, fam)
    nf = g.NearField(d, d, sp, "[1/r]", sp)
    nf.compute(s)
    n = sp.free_count()
    A = torch.zeros(n * n, dtype=torch.complex128, device="cuda")
    nf.apply(A.data_ptr(), n, s)
    r, c, v = nf.triplets()
    torch.cuda.synchronize()
    print(f"nearfield {fam} g{gauss}: {len(v)} entries, sum={float(np.sum(v)):.6e}")

d = g.make_domain(mesh, 3)
pts, w, _ = g.quadrature(d)
pts = np.asarray(pts)
q = np.asarray(w) * g.complex_normal(4, len(w))
qd = torch.tensor(q, device="cuda")
for tgt, label in ((pts, "sym"), (pts[: len(pts) // 3] * 1.5, "general")):
    gp = g.GreenPlan(tgt, pts, g.green_kernel("[exp(ikr)/r]", k))
    y = torch.empty(len(tgt), dtype=torch.complex128, device="cuda")
    for prec in (g.FP64, g.FP32):
        gp.matvec(qd.data_ptr(), y.data_ptr(), prec, s)
        torch.cuda.synchronize()
        print(f"green {label} prec={prec}: |y|={float(y.abs().sum()):.6e}")

sp = g.make_fem(mesh, "P1")
ev = g.GalerkinEvaluator(d, d, sp, g.green_kernel("[exp(ikr)/r]", k), sp)
blk = np.asarray(ev.eval(list(range(0, 40, 3)), list(range(5, 60, 7))))
print(f"block eval: {blk.shape} |B|={float(np.abs(blk).sum()):.6e}")
print("sanitize_probe: done")
