"""F_analytic probe: the reference formula of
analytic_triangle_integrals (kernels.cpp:151-207, libdevice) evaluated on the
(triangle, point) mix regularize produces on BASELINE cfg 3: the y triangle of
every near element pair against the 7-point rule points of the x triangle's
sub-cells down to depth 2 (the calls accurate_adaptive makes, assembly.cpp:
548-605).  Run under
  ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,\
smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum \
      -k regex:k_probe_analytic python scripts/fanalytic_probe.py
and divide by the printed call count: flops per call = 2 DFMA + DMUL + DADD."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_00995_b200 as g  # noqa: E402
from tests._support import load_oracle  # noqa: E402

o = load_oracle()
v, e = o.perturb_radial(*o.build_sphere(10242, 1.0), 2, 0.02)
v, e = np.asarray(v), np.asarray(e)
hbar = o.edge_stats(v, e)[2]
pairs = np.asarray(o.near_pairs(v, e, v, e, 0, hbar))
rng = np.random.default_rng(3)
sel = pairs[rng.choice(len(pairs), 4096, replace=False)]
b7, _ = o.rule(7)
b7 = np.asarray(b7).reshape(7, 3)
# sub-cells down to depth 2: corners in barycentric coordinates of the x triangle
cells = [np.eye(3)]
for _ in range(2):
    nxt = []
    for c in cells:
        m01, m12, m20 = (c[0] + c[1]) / 2, (c[1] + c[2]) / 2, (c[2] + c[0]) / 2
        nxt += [np.array([c[0], m01, m20]), np.array([m01, c[1], m12]), np.array([m20, m12, c[2]]),
                np.array([m01, m12, m20])]
    cells = cells + nxt
tri, pts = [], []
for ex, ey in sel:
    X = v[e[ex]]
    for c in cells[::3]:
        bary = b7 @ c  # 7 rule points of the sub-cell, barycentric in the x triangle
        for bq in bary:
            tri.append(v[e[ey]].ravel())
            pts.append(bq @ X)
tri, pts = np.asarray(tri), np.asarray(pts)
n = len(pts)
td = torch.tensor(tri.ravel(), device="cuda")
pd = torch.tensor(pts.ravel(), device="cuda")
out = torch.empty(4 * n, dtype=torch.float64, device="cuda")
g.diag_probe_analytic(n, td.data_ptr(), pd.data_ptr(), n, out.data_ptr(), 0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.diag_probe_analytic(n, td.data_ptr(), pd.data_ptr(), n, out.data_ptr(), 0)
e1.record()
torch.cuda.synchronize()
r = out.cpu().numpy().reshape(n, 4)
ref = np.array([o.analytic(tri[i, :3], tri[i, 3:6], tri[i, 6:], pts[i])[0] for i in range(0, n, max(1, n // 2000))])
print("calls", n, "ms", e0.elapsed_time(e1), "newton max rel vs oracle",
      float(np.max(np.abs(r[:: max(1, n // 2000), 0] - ref) / np.abs(ref))))
