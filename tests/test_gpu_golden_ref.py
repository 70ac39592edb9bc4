"""GPU against the REFERENCE-HELD vectors (tests/golden/golden_ref_v1.npz:
outputs of the reference's own assembly.cpp / kernels.cpp / oracles.cpp,
compiled unchanged against the Eigen-API shim; tests/golden/make_golden_ref.py).
The device path (plans, near field, point rows, panel) reproduces the
reference's numbers within the north-star bar (1e-10 relative Frobenius)
without the reference or the oracle at run time."""
import os

import numpy as np
import pytest

from tests._support import rel_fro

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
TOL = 1e-10


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(HERE, "golden", "golden_ref_v1.npz"))


def _mesh(galerk, gold, tag):
    return galerk.Mesh(gold[f"{tag}_vertices"], gold[f"{tag}_elements"])


def _sorted(r, c, v):
    r, c, v = map(np.asarray, (r, c, v))
    o = np.lexsort((r, c))
    return r[o], c[o], v[o]


@pytest.mark.parametrize("key,g,fam,name", [("A_l2_p1_r3_helm", 3, "P1", "[exp(ikr)/r]"),
                                            ("A_l2_p1_r3_lap", 3, "P1", "[1/r]"),
                                            ("A_l2_p0_r7_helm", 7, "P0", "[exp(ikr)/r]"),
                                            ("A_l2_p1_r7_helm", 7, "P1", "[exp(ikr)/r]")])
def test_bem_dense_vs_reference(galerk, gold, key, g, fam, name):
    m = _mesh(galerk, gold, "l2")
    dom, sp = galerk.make_domain(m, g), galerk.make_fem(m, fam)
    k = 0.0 if name == "[1/r]" else float(gold["l2_k"])
    A = galerk.bem_dense(dom, dom, sp, galerk.green_kernel(name, k), sp)
    assert rel_fro(A, gold[key]) <= TOL
    if name == "[1/r]":
        assert np.all(A.imag == 0.0)


def test_mixed_and_naive_vs_reference(galerk, gold):
    mx, my = _mesh(galerk, gold, "l2"), _mesh(galerk, gold, "l1")
    A = galerk.bem_dense(galerk.make_domain(mx, 1), galerk.make_domain(my, 3), galerk.make_fem(mx, "P1"),
                         galerk.green_kernel("[exp(ikr)/r]", 2.5), galerk.make_fem(my, "P0"))
    assert rel_fro(A, gold["A_mixed_p1r1_p0r3"]) <= TOL
    m0 = _mesh(galerk, gold, "l0")
    d0, s0 = galerk.make_domain(m0, 3), galerk.make_fem(m0, "P1")
    B = galerk.bem_dense(d0, d0, s0, galerk.green_kernel("[exp(ikr)/r]", 2.0), s0)
    # the reference's own structural pin: bem_dense == naive_bem to 1e-13 (test_assembly.cpp:159-180)
    assert np.abs(B - gold["naive_l0_p1"]).max() <= 1e-13 * np.abs(gold["naive_l0_p1"]).max()


@pytest.mark.parametrize("tag,g,fam", [("p1r3", 3, "P1"), ("p0r7", 7, "P0"), ("p0r3", 3, "P0")])
def test_regularize_vs_reference(galerk, gold, tag, g, fam):
    m = _mesh(galerk, gold, "l2")
    dom, sp = galerk.make_domain(m, g), galerk.make_fem(m, fam)
    nf = galerk.NearField(dom, dom, sp, "[1/r]", sp)
    nf.compute(0)
    r, c, v = _sorted(*nf.triplets())
    gr, gc, gv = _sorted(gold[f"nf_{tag}_rows"], gold[f"nf_{tag}_cols"], gold[f"nf_{tag}_vals"])
    assert np.array_equal(r, gr) and np.array_equal(c, gc)
    assert rel_fro(v, gv) <= TOL


def test_radiation_vs_reference(galerk, gold):
    m = _mesh(galerk, gold, "l2")
    dom, sp = galerk.make_domain(m, 3), galerk.make_fem(m, "P1")
    R = galerk.radiation_dense(gold["rad_points"], dom, galerk.green_kernel("[exp(ikr)/r]", float(gold["l2_k"])), sp)
    assert rel_fro(R, gold["rad_p1_r3"]) <= TOL
    colptr, rows, vals, shape = galerk.regularize_radiation(gold["radnf_points"], dom, "[1/r]", sp)
    cols = np.repeat(np.arange(shape[1]), np.diff(colptr))
    r, c, v = _sorted(rows, cols, vals)
    gr, gc, gv = _sorted(gold["radnf_p1_rows"], gold["radnf_p1_cols"], gold["radnf_p1_vals"])
    assert np.array_equal(r, gr) and np.array_equal(c, gc) and rel_fro(v, gv) <= TOL


def test_evaluate_blocks_vs_reference(galerk, gold):
    X, Y = gold["eval_X"], gold["eval_Y"]
    eps = 1e-12 * float(np.linalg.norm(np.vstack([X, Y]).max(axis=0) - np.vstack([X, Y]).min(axis=0)))
    K = galerk.evaluate_blocks(X, Y, galerk.green_kernel("[exp(ikr)/r]", 7.5), eps, True)
    assert rel_fro(K, gold["eval_K"]) <= 1e-13
    assert np.array_equal(K == 0, gold["eval_K"] == 0)
