"""Regenerates tests/golden/golden_ref_v1.npz from the REFERENCE'S OWN CODE
(test infrastructure): /root/reference/proj/src/{mesh,quadrature,kernels,
femspace,assembly}.cpp and tests/support/oracles.cpp compiled unchanged
against the Eigen-API shim (oracle/_ref, oracle/Makefile `ref`).  These are
reference-held vectors: the GPU suite checks the device against them
(tests/test_gpu_golden_ref.py) and the CPU suite checks the oracle against
them, neither needing /root/reference at run time.

    python tests/golden/make_golden_ref.py
"""
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from tests._support import load_ref  # noqa: E402

P0, P1 = 0, 1


def build(ref):
    out = {}
    v, e = ref.build_sphere(162, 1.0)
    out["l2_vertices"], out["l2_elements"] = v, e
    hbar = ref.edge_stats(v, e)[2]
    k = 2 * math.pi / (10 * hbar)
    out["l2_k"] = np.array(k)
    # bem_dense (assembly.cpp:313-320): P1/P0, rules 3 and 7, Helmholtz / Laplace
    out["A_l2_p1_r3_helm"] = ref.bem_dense(v, e, 3, P1, v, e, 3, P1, "[exp(ikr)/r]", k)
    out["A_l2_p1_r3_lap"] = ref.bem_dense(v, e, 3, P1, v, e, 3, P1, "[1/r]", 0.0)
    out["A_l2_p0_r7_helm"] = ref.bem_dense(v, e, 7, P0, v, e, 7, P0, "[exp(ikr)/r]", k)
    out["A_l2_p1_r7_helm"] = ref.bem_dense(v, e, 7, P1, v, e, 7, P1, "[exp(ikr)/r]", k)
    # mixed: P1 test on L2, P0 trial on L1 (non-symmetric), rule 1 x rule 3
    v1, e1 = ref.build_sphere(42, 1.3)
    out["l1_vertices"], out["l1_elements"] = v1, e1
    out["A_mixed_p1r1_p0r3"] = ref.bem_dense(v, e, 1, P1, v1, e1, 3, P0, "[exp(ikr)/r]", 2.5)
    # naive_bem (tests/support/oracles.cpp:332-360) on the icosahedron
    v0, e0 = ref.build_sphere(12, 1.0)
    out["l0_vertices"], out["l0_elements"] = v0, e0
    out["naive_l0_p1"] = ref.naive_bem(v0, e0, 3, P1, v0, e0, 3, P1, "[exp(ikr)/r]", 2.0)
    # regularize (assembly.cpp:609-697) P1 and P0, rules 3 / 7
    for fam, g, tag in ((P1, 3, "p1r3"), (P0, 7, "p0r7"), (P0, 3, "p0r3")):
        r, c, val = ref.regularize(v, e, g, fam, v, e, g, fam, "[1/r]")
        out[f"nf_{tag}_rows"] = np.asarray(r, dtype=np.int32)
        out[f"nf_{tag}_cols"] = np.asarray(c, dtype=np.int32)
        out[f"nf_{tag}_vals"] = np.asarray(val)
    # radiation_dense (assembly.cpp:334-341) and regularize_radiation (:699-750)
    # at points off the surface (on-vertex collocation is NaN in the reference)
    rng = np.random.default_rng(5)
    pts = rng.normal(size=(40, 3))
    pts = pts / np.linalg.norm(pts, axis=1, keepdims=True) * rng.uniform(0.5, 2.0, size=(40, 1))
    out["rad_points"] = pts
    out["rad_p1_r3"] = ref.radiation_dense(pts, v, e, 3, P1, "[exp(ikr)/r]", k)
    cen = v[e].mean(axis=1)[:50] * 1.001  # 0.1% outside the surface, near the centroids
    out["radnf_points"] = cen
    r, c, val = ref.regularize_radiation(cen, v, e, 3, P1, "[1/r]")
    out["radnf_p1_rows"], out["radnf_p1_cols"] = np.asarray(r, dtype=np.int32), np.asarray(c, dtype=np.int32)
    out["radnf_p1_vals"] = np.asarray(val)
    # evaluate_blocks (kernels.cpp:76-131) with coincident pairs masked
    X = rng.normal(size=(60, 3))
    Y = np.vstack([rng.normal(size=(40, 3)), X[:4]])
    out["eval_X"], out["eval_Y"] = X, Y
    out["eval_K"] = ref.evaluate("[exp(ikr)/r]", 7.5, X, Y, True, -1.0)
    return out


if __name__ == "__main__":
    ref = load_ref()
    if ref is None:
        sys.exit("oracle/_ref is not built and /root/reference is absent")
    d = build(ref)
    path = os.path.join(HERE, "golden_ref_v1.npz")
    np.savez_compressed(path, **d)
    print(path, os.path.getsize(path), "bytes:", sorted(d))
