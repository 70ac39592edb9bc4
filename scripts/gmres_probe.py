"""How far the device GMRES history tracks the numpy restatement (MGS both)."""
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import linsolve_oracle  # noqa: E402

import paper_1804_00995_b200 as g  # noqa: E402
from tests._support import sphere_problem  # noqa: E402

for name, k, restart, shifted in (("[exp(ikr)/r]", 3.0, 50, True), ("[exp(ikr)/r]", 6.0, 10, True),
                                  ("[1/r]", 0.0, 30, True), ("[exp(ikr)/r]", 3.0, 50, False)):
    m, dom, sp, _ = sphere_problem(g, 642, 3, "P1")
    S = g.bem_dense(dom, dom, sp, g.green_kernel(name, k), sp) / (4 * math.pi)
    if shifted:
        S = S + np.abs(np.diag(S)).mean() * np.eye(S.shape[0])
    rng = np.random.default_rng(11)
    b = rng.normal(size=642) + 1j * rng.normal(size=642)
    n = S.shape[0]
    Ad = torch.tensor(np.asfortranarray(S).T.copy(), dtype=torch.complex128, device="cuda")
    bd = torch.tensor(b, dtype=torch.complex128, device="cuda")
    xd = torch.empty(n, dtype=torch.complex128, device="cuda")
    info = g.gmres(Ad.data_ptr(), n, n, bd.data_ptr(), xd.data_ptr(), 1e-8, restart, 2000)
    xo, io = linsolve_oracle.gmres(lambda v: S @ v, b, 1e-8, restart, 2000)
    h, ho = np.array(info["history"]), np.array(io["history"])
    ne = min(len(h), len(ho))
    rel = np.abs(h[:ne] - ho[:ne]) / np.abs(ho[:ne])
    first_bad = int(np.argmax(rel > 1e-8)) if np.any(rel > 1e-8) else ne
    print(f"{name} k={k} restart={restart} shifted={shifted}: iters dev {info['iterations']} oracle {io['iterations']}, "
          f"history agrees to 1e-8 for {first_bad}/{ne} entries, max rel over first 10 {rel[:10].max():.2e}")
