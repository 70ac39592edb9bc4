"""Pin the oracle (and the product's host tables) to the REFERENCE'S OWN CODE.

oracle/_ref is /root/reference/proj/src/{mesh,quadrature,kernels}.cpp compiled
unchanged against a minimal Eigen-API shim (oracle/eigen_shim, oracle/Makefile
`ref`; Eigen itself is absent here).  Everything the dense assembly and the
matrix-free matvec read from those files must agree BIT FOR BIT:
  build_sphere (mesh.cpp:253-309), edge_stats (:535-567), element_measure
  (:47-69), the triangle rules and quadrature() (quadrature.cpp:40-75,
  167-189), singular_guard_radius (kernels.cpp:14-19), Kernel::green +
  evaluate_blocks with the distance mask and its raising path
  (kernels.cpp:21-54, 76-131), analytic_triangle_integrals (kernels.cpp:151-207).
The oracle's bem_product / regularize are then built on pinned leaves; their
own structure is pinned by test_oracle_pins.py (the reference's tests).
"""
import numpy as np
import pytest

from tests._support import load_ref

ref = load_ref()
pytestmark = pytest.mark.skipif(ref is None, reason="oracle/_ref not built and /root/reference absent")

SIZES = (12, 42, 162, 642, 2562, 10242)


@pytest.mark.parametrize("n", SIZES + (40962,))
def test_build_sphere_bitwise(oracle, galerk, n):
    v, e = ref.build_sphere(n, 1.0)
    vo, eo = oracle.build_sphere(n, 1.0)
    assert np.array_equal(v, vo) and np.array_equal(e, eo)
    m = galerk.build_sphere(n, 1.0)
    assert np.array_equal(v, np.asarray(m.vertices)) and np.array_equal(e, np.asarray(m.elements))
    assert ref.edge_stats(v, e) == oracle.edge_stats(v, e)
    s = galerk.edge_stats(m)
    assert (s.min_len, s.max_len, s.mean_len, s.std_len) == ref.edge_stats(v, e)
    assert ref.element_measures(v, e) == oracle.element_measures(v, e)


@pytest.mark.parametrize("g", (1, 3, 7))
@pytest.mark.parametrize("n", (12, 642, 10242))
def test_rules_and_quadrature_bitwise(oracle, galerk, n, g):
    assert ref.rule(g) == tuple(list(np.ravel(x)) for x in oracle.rule(g))
    v, e = ref.build_sphere(n, 1.0)
    p, w, el = ref.quadrature(v, e, g)
    po, wo, elo = oracle.quadrature(v, e, g)
    assert np.array_equal(p, po) and np.array_equal(w, wo) and np.array_equal(el, elo)
    m = galerk.build_sphere(n, 1.0)
    pg, wg, elg = galerk.quadrature(galerk.make_domain(m, g))
    assert np.array_equal(p, np.asarray(pg)) and np.array_equal(w, np.asarray(wg))


def test_perturbed_mesh_quadrature_bitwise(oracle):
    # cfg 3 mesh (radially perturbed L5): the perturbation is the repo's own
    # seeded generator; everything downstream of it is the reference's code
    v, e = oracle.perturb_radial(*oracle.build_sphere(10242, 1.0), 2, 0.02)
    assert ref.edge_stats(v, e) == oracle.edge_stats(v, e)
    for g in (1, 3, 7):
        p, w, _ = ref.quadrature(v, e, g)
        po, wo, _ = oracle.quadrature(v, e, g)
        assert np.array_equal(p, po) and np.array_equal(w, wo)


@pytest.mark.parametrize("name,k", [("[exp(ikr)/r]", 3.7), ("[exp(ikr)/r]", 66.8), ("[1/r]", 5.0),
                                    ("[exp(ikr)/r]", 0.0)])
def test_evaluate_blocks_bitwise(oracle, name, k):
    rng = np.random.default_rng(7)
    X = rng.normal(size=(70, 3))
    Y = np.vstack([rng.normal(size=(50, 3)), X[:5]])  # coincident pairs hit the mask
    assert ref.singular_guard_radius(X, Y) == oracle.singular_guard_radius(X, Y)
    a = ref.evaluate(name, k, X, Y, True, -1.0)
    b = oracle.evaluate(name, k, X, Y, True, -1.0)
    assert np.array_equal(a, b)
    assert np.count_nonzero(a == 0) == 5
    assert ref.kernel_info(name, k)[1] == (0.0 if name == "[1/r]" else k)


def test_evaluate_blocks_raising_path(oracle):
    # mask=false on a coincident pair raises with the pair index (kernels.cpp:104-108)
    X = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0]])
    with pytest.raises(RuntimeError, match=r"\(1,0\)") as e_ref:
        ref.evaluate("[exp(ikr)/r]", 2.0, X, X[1:], False, -1.0)
    with pytest.raises(RuntimeError, match=r"\(1,0\)") as e_or:
        oracle.evaluate("[exp(ikr)/r]", 2.0, X, X[1:], False, -1.0)
    assert str(e_ref.value).split(", r=")[0] == str(e_or.value).split(", r=")[0]


def test_unknown_kernel_name_message(oracle):
    with pytest.raises(ValueError) as a:
        ref.kernel_info("[log r]", 1.0)
    with pytest.raises(ValueError) as b:
        oracle.evaluate("[log r]", 1.0, np.zeros((1, 3)), np.ones((1, 3)), True, -1.0)
    assert str(a.value) == str(b.value)


def test_analytic_triangle_integrals_bitwise(oracle):
    rng = np.random.default_rng(11)
    for i in range(3000):
        a, b, c, x = rng.normal(size=(4, 3))
        if i % 3 == 0:  # in-plane points (inside and outside the triangle)
            s, t = rng.uniform(-0.5, 1.2, size=2)
            x = a + s * (b - a) + t * (c - a)
        if i % 7 == 0:  # near a vertex / an edge
            x = a + 1e-6 * rng.normal(size=3) if i % 2 else 0.5 * (a + b) + 1e-9 * rng.normal(size=3)
        assert repr(ref.analytic(a, b, c, x)) == repr(oracle.analytic(a, b, c, x)), i
    # degenerate triangle raises the reference's message
    z = [0.0, 0.0, 0.0]
    with pytest.raises(ValueError, match="degenerate triangle"):
        ref.analytic(z, [1.0, 0, 0], [2.0, 0, 0], [0.0, 1.0, 0])
    with pytest.raises(ValueError, match="degenerate triangle"):
        oracle.analytic(z, [1.0, 0, 0], [2.0, 0, 0], [0.0, 1.0, 0])
