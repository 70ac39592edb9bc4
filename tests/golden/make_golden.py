"""Regenerates tests/golden/golden_v1.npz from the CPU oracle (test infrastructure).

The reference itself cannot be built here (no Eigen), so these fixtures are
outputs of the oracle (pinned to the reference's own known-answer tests in
tests/test_oracle_pins.py).  Committing them freezes the oracle's outputs: the
CPU suite checks the oracle still reproduces them bit for bit, and the GPU
suite checks the device against them without re-running the oracle.

    python tests/golden/make_golden.py
"""
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from tests._support import load_oracle  # noqa: E402

P0, P1 = 0, 1


def build(oracle):
    out = {}
    v, e = oracle.build_sphere(162, 1.0)
    v, e = np.asarray(v), np.asarray(e)
    out["l2_vertices"], out["l2_elements"] = v, e
    hbar = oracle.edge_stats(v, e)[2]
    k = 2 * math.pi / (10 * hbar)
    out["l2_k"] = np.array(k)
    # cfg-2-like: Helmholtz P1 3-point, the full matrix
    out["A_l2_p1_helm"] = oracle.bem_dense(v, e, 3, P1, v, e, 3, P1, "[exp(ikr)/r]", k)
    # cfg-1-like: Laplace P1 3-point
    out["A_l2_p1_lap"] = oracle.bem_dense(v, e, 3, P1, v, e, 3, P1, "[1/r]", 0.0)
    # cfg-3-like: P0, the new 6-point rule, on a radially perturbed L1 sphere (seed 2)
    v1, e1 = oracle.build_sphere(42, 1.0)
    v1, e1 = oracle.perturb_radial(np.asarray(v1), np.asarray(e1), 2, 0.02)
    v1, e1 = np.asarray(v1), np.asarray(e1)
    out["l1p_vertices"], out["l1p_elements"] = v1, e1
    out["A_l1p_p0_rule6_helm"] = oracle.bem_dense(v1, e1, 6, P0, v1, e1, 6, P0, "[exp(ikr)/r]", 3.0)
    # near-field correction (regularize), P1 x P1 and P0 x P0 on L2
    for fam, tag in ((P1, "p1"), (P0, "p0")):
        r, c, val, _ = oracle.regularize(v, e, 3, fam, v, e, 3, fam, "[1/r]", threads=4)
        out[f"nf_l2_{tag}_rows"] = np.asarray(r, dtype=np.int32)
        out[f"nf_l2_{tag}_cols"] = np.asarray(c, dtype=np.int32)
        out[f"nf_l2_{tag}_vals"] = np.asarray(val)
    # matrix-free Green matvec on the L2 Gauss points (targets = sources), seed 4 charges
    pts, w, _ = oracle.quadrature(v, e, 3)
    pts = np.asarray(pts)
    u = np.asarray(oracle.uniform01_stream(4, 2 * len(w)))
    out["green_l2_points"] = pts
    out["green_l2_q"] = np.asarray(w) * (u[0::2] + 1j * u[1::2])
    lo, hi = pts.min(axis=0), pts.max(axis=0)
    eps = 1e-12 * float(np.linalg.norm(hi - lo))
    out["green_l2_eps"] = np.array(eps)
    out["green_l2_y"] = np.asarray(oracle.green_matvec("[exp(ikr)/r]", k, pts, pts, out["green_l2_q"], eps,
                                                       list(range(len(pts))), 4))
    return out


if __name__ == "__main__":
    o = load_oracle()
    d = build(o)
    path = os.path.join(HERE, "golden_v1.npz")
    np.savez_compressed(path, **d)
    print(path, os.path.getsize(path), "bytes:", sorted(d))
