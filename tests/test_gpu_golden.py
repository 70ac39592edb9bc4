"""GPU vs the committed golden fixtures (tests/golden/golden_v1.npz): the
device reproduces the frozen oracle outputs without running the oracle."""
import os

import numpy as np
import pytest

from tests._support import rel_fro

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
TOL = 1e-10


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(HERE, "golden", "golden_v1.npz"))


def test_dense_matrices(galerk, golden):
    m = galerk.build_sphere(162, 1.0)
    dom = galerk.make_domain(m, 3)
    p1 = galerk.make_fem(m, "P1")
    k = float(golden["l2_k"])
    A = galerk.bem_dense(dom, dom, p1, galerk.green_kernel("[exp(ikr)/r]", k), p1)
    assert rel_fro(A, golden["A_l2_p1_helm"]) <= TOL
    L = galerk.bem_dense(dom, dom, p1, galerk.green_kernel("[1/r]", 0.0), p1)
    assert rel_fro(L, golden["A_l2_p1_lap"]) <= TOL and np.all(L.imag == 0.0)
    m1 = galerk.perturb_radial(galerk.build_sphere(42, 1.0), 2, 0.02)
    d1 = galerk.make_domain(m1, 6)
    p0 = galerk.make_fem(m1, "P0")
    B = galerk.bem_dense(d1, d1, p0, galerk.green_kernel("[exp(ikr)/r]", 3.0), p0)
    assert rel_fro(B, golden["A_l1p_p0_rule6_helm"]) <= TOL


@pytest.mark.parametrize("fam", ["p1", "p0"])
def test_near_field(galerk, golden, fam):
    m = galerk.build_sphere(162, 1.0)
    dom = galerk.make_domain(m, 3)
    sp = galerk.make_fem(m, fam.upper())
    nf = galerk.NearField(dom, dom, sp, "[1/r]", sp)
    nf.compute(0)
    r, c, v = nf.triplets()
    o = np.lexsort((np.asarray(r), np.asarray(c)))
    go = np.lexsort((golden[f"nf_l2_{fam}_rows"], golden[f"nf_l2_{fam}_cols"]))
    assert np.array_equal(np.asarray(r)[o], golden[f"nf_l2_{fam}_rows"][go])
    assert np.array_equal(np.asarray(c)[o], golden[f"nf_l2_{fam}_cols"][go])
    assert rel_fro(np.asarray(v)[o], golden[f"nf_l2_{fam}_vals"][go]) <= TOL


def test_green_matvec(galerk, golden):
    import torch

    pts, q = golden["green_l2_points"], golden["green_l2_q"]
    plan = galerk.GreenPlan(pts, pts, galerk.green_kernel("[exp(ikr)/r]", float(golden["l2_k"])))
    assert plan.info()["eps"] == float(golden["green_l2_eps"])
    qd = torch.tensor(q, device="cuda")
    y = torch.empty(len(pts), dtype=torch.complex128, device="cuda")
    plan.matvec(qd.data_ptr(), y.data_ptr(), galerk.FP64, 0)
    torch.cuda.synchronize()
    assert rel_fro(y.cpu().numpy(), golden["green_l2_y"]) <= TOL
