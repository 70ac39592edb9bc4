"""Pin the CPU oracle to the reference's own known-answer tests.

The reference (/root/reference/proj) cannot be built here (no Eigen, no
doctest), so the oracle is pinned by porting the reference's tests for this
path, with the reference's own tolerances:
  test_mesh.cpp:75-84, test_quadrature.cpp:32-85,160-166,
  test_femspace.cpp:62-71,86-94, test_kernels.cpp:31-65,98-182,
  test_assembly.cpp:136-260.
"""
import math

import numpy as np
import pytest

from tests._support import rel_fro

P0, P1 = 0, 1


def single_triangle(scale=1.0):
    v = np.array([[0, 0, 0], [scale, 0, 0], [0, scale, 0]], dtype=np.float64)
    e = np.array([[0, 1, 2]], dtype=np.int32)
    return v, e


# ---- test_mesh.cpp:75-84 ----------------------------------------------------
def test_build_sphere_counts_and_area(oracle):
    v, e = oracle.build_sphere(12, 1.0)
    assert v.shape == (12, 3) and e.shape == (20, 3)
    v, e = oracle.build_sphere(1000, 1.0)
    assert v.shape[0] == 2562
    area = sum(oracle.element_measures(v, e))
    assert abs(area - 4 * math.pi) / (4 * math.pi) < 0.005
    with pytest.raises(ValueError):
        oracle.build_sphere(5, 1.0)


def test_sphere_configs_match_survey_table(oracle):
    # vertex/triangle counts and mean edge lengths.
    for n, ne, hbar in ((642, 1280, 0.15008), (10242, 20480, 0.037593)):
        v, e = oracle.build_sphere(n, 1.0)
        assert v.shape[0] == n and e.shape[0] == ne
        assert abs(oracle.edge_stats(v, e)[2] - hbar) < 1e-5
    # outward orientation
    v, e = oracle.build_sphere(642, 1.0)
    a, b, c = v[e[:, 0]], v[e[:, 1]], v[e[:, 2]]
    assert np.all(np.einsum("ij,ij->i", np.cross(b - a, c - a), a + b + c) > 0)


# ---- test_quadrature.cpp ------------------------------------------------------
def test_rule_ids_validated(oracle):
    with pytest.raises(ValueError, match="1,3,7"):
        oracle.rule(5)


@pytest.mark.parametrize("g", [1, 3, 6, 7])
def test_weights_sum_to_measure(oracle, g):
    v, e = oracle.build_sphere(642, 1.0)
    pts, w, elem = oracle.quadrature(v, e, g)
    assert abs(sum(w) - sum(oracle.element_measures(v, e))) <= 1e-12 * sum(w)
    assert min(w) > 0
    assert elem == [i // g for i in range(len(elem))]  # contiguity pin :160-166


@pytest.mark.parametrize("g,degree", [(1, 1), (3, 2), (6, 4), (7, 5)])
def test_degree_exactness(oracle, g, degree):
    v, e = single_triangle()
    pts, w, _ = oracle.quadrature(v, e, g)
    for a in range(degree + 1):
        for b in range(degree + 1 - a):
            got = sum(wi * p[0] ** a * p[1] ** b for wi, p in zip(w, pts))
            exp = oracle.simplex_monomial(2, a, b, 0)
            assert abs(got - exp) <= 1e-12 * max(1.0, abs(exp)), (a, b)
    if g == 6:  # the new rule is exactly degree 4: x^5 is not integrated exactly
        got = sum(wi * p[0] ** 5 for wi, p in zip(w, pts))
        assert abs(got - oracle.simplex_monomial(2, 5, 0, 0)) > 1e-6


def test_three_point_rule_is_edge_midpoints(oracle):
    bary, w = oracle.rule(3)
    assert sorted(map(tuple, bary)) == sorted([(0.5, 0.5, 0.0), (0.0, 0.5, 0.5), (0.5, 0.0, 0.5)])
    # on a closed mesh each location is shared by exactly two triangles (SURVEY trap 1)
    v, e = oracle.build_sphere(642, 1.0)
    pts, _, _ = oracle.quadrature(v, e, 3)
    _, counts = np.unique(np.asarray(pts), axis=0, return_counts=True)
    assert np.all(counts == 2)


# ---- test_femspace.cpp ----------------------------------------------------------
def test_p1_centroid_row_and_p0_indicator(oracle):
    v, e = single_triangle()
    start, dof, val = oracle.eval_rows(v, e, P1, 1)
    assert start == [0, 3] and dof == [0, 1, 2]
    assert np.allclose(val, 1 / 3, rtol=1e-14)
    v, e = oracle.build_sphere(42, 1.0)
    start, dof, val = oracle.eval_rows(v, e, P0, 3)
    assert dof == [k // 3 for k in range(3 * 80)] and set(val) == {1.0}
    # P1 midpoint rule: exactly 2 nonzeros per row, 0.5 each
    start, dof, val = oracle.eval_rows(v, e, P1, 3)
    assert np.all(np.diff(start) == 2) and set(val) == {0.5}


# ---- test_kernels.cpp -------------------------------------------------------------
def test_scalar_kernels(oracle, rng):
    v = oracle.evaluate("[1/r]", 0.0, np.zeros((1, 3)), np.array([[0, 0, 2.0]]))
    assert abs(v[0, 0].real - 0.5) <= 1e-15 and v[0, 0].imag == 0.0
    X = rng.uniform(-2, 2, (4, 3))
    Y = rng.uniform(-2, 2, (3, 3)) + [5, 0, 0]
    a = oracle.evaluate("[exp(ikr)/r]", 0.0, X, Y)
    b = oracle.evaluate("[1/r]", 0.0, X, Y)
    assert np.abs(a - b).max() < 1e-15
    same = np.array([[1.0, 2.0, 3.0]])
    with pytest.raises(RuntimeError, match=r"\(0,0\)"):
        oracle.evaluate("[1/r]", 0.0, same, same)
    with pytest.raises(ValueError):
        oracle.evaluate("[foo]", 1.0, X, Y)


def test_reciprocity(oracle, rng):
    for name, k in (("[exp(ikr)/r]", 3.0), ("[1/r]", 0.0)):
        X = rng.uniform(-1, 1, (5, 3))
        Y = rng.uniform(-1, 1, (6, 3)) + [3, 0, 0]
        a = oracle.evaluate(name, k, X, Y)
        b = oracle.evaluate(name, k, Y, X)
        assert np.abs(a - b.T).max() < 1e-14


def test_analytic_specific_cases(oracle):
    a, b, c = (0, 0, 0), (1, 0, 0), (0, 1, 0)
    cen = (1 / 3, 1 / 3, 0)
    assert abs(oracle.analytic(a, b, c, cen)[0] - oracle.newton_oracle(a, b, c, cen, 1e-11)) <= 1e-8 * 1.5
    far = (60.0, 50.0, 60.0)
    tn = oracle.analytic(a, b, c, far)
    dist = np.linalg.norm(np.subtract(far, cen))
    assert abs(tn[0] - 0.5 / dist) < 1e-4 * (0.5 / dist)
    g = np.array(tn[1])
    assert abs(g @ (np.subtract(far, cen)) / np.linalg.norm(g) / dist - 1) < 1e-4
    s3 = math.sqrt(3.0)
    ts = oracle.analytic((1, 0, 0), (-0.5, s3 / 2, 0), (-0.5, -s3 / 2, 0), (0, 0, 0.7))
    assert abs(ts[1][0]) < 1e-12 and abs(ts[1][1]) < 1e-12
    with pytest.raises(ValueError):
        oracle.analytic(a, b, a, cen)


def test_analytic_random_configurations(oracle):
    rng = np.random.default_rng(7)
    inside = 0
    trial = 0
    while trial < 100:
        a, b, c = (rng.uniform(-1, 1, 3) for _ in range(3))
        if np.linalg.norm(np.cross(b - a, c - a)) < 0.05:
            continue
        mode = trial % 4
        if mode == 0:
            r1, r2 = 0.2 + 0.2 * rng.uniform(-1, 1), 0.2 + 0.2 * rng.uniform(-1, 1)
            x = a + r1 * (b - a) + r2 * (c - a)
            inside += 1
        elif mode == 1:
            x = rng.uniform(-2, 2, 3)
        elif mode == 2:
            n = np.cross(b - a, c - a)
            n /= np.linalg.norm(n)
            x = (a + b + c) / 3 + 0.01 * n + 0.3 * (b - a)
        else:
            x = rng.uniform(-5, 5, 3)
        tn = oracle.analytic(a, b, c, x)
        nw = oracle.newton_oracle(a, b, c, x, 1e-11)
        assert abs(tn[0] - nw) <= 1e-8 * max(1.0, abs(nw))
        mo = np.array(oracle.newton_moment_oracle(a, b, c, x, 1e-11))
        assert np.linalg.norm(np.array(tn[2]) - mo) <= 1e-7 * max(1.0, np.linalg.norm(mo))
        n = np.cross(b - a, c - a)
        n /= np.linalg.norm(n)
        if abs((x - a) @ n) > 0.2:
            gr = np.array(oracle.newton_grad_oracle(a, b, c, x, 1e-12))
            assert np.linalg.norm(np.array(tn[1]) - gr) <= 1e-7 * max(1.0, np.linalg.norm(gr))
        trial += 1
    assert inside >= 20


def test_normal_jump_of_gradient(oracle):
    a, b, c = (0, 0, 0), (1, 0, 0), (0, 1, 0)
    up = oracle.analytic(a, b, c, (0.3, 0.3, 1e-9))[1]
    dn = oracle.analytic(a, b, c, (0.3, 0.3, -1e-9))[1]
    assert abs((up[2] - dn[2]) - 4 * math.pi) <= 1e-6 * 4 * math.pi
    assert abs(up[0] - dn[0]) <= 1e-6 * abs(dn[0]) and abs(up[1] - dn[1]) <= 1e-6 * abs(dn[1])


# ---- test_assembly.cpp ----------------------------------------------------------
def test_bem_dense_basics(oracle):
    v1, e1 = single_triangle(1.0)
    v2, e2 = single_triangle(2.0)
    v2[:, 2] += 5.0
    a = oracle.bem_dense(v1, e1, 3, P0, v2, e2, 3, P0, "__ones__", 0.0)
    assert abs(a[0, 0].real - 0.5 * 2.0) <= 1e-13 * 2.0
    v, e = oracle.build_sphere(42, 1.0)
    s = oracle.bem_dense(v, e, 3, P1, v, e, 3, P1, "[1/r]", 0.0)
    assert np.abs(s - s.T).max() <= 1e-12 * np.abs(s).max()


def test_bem_dense_equals_naive_oracle(oracle):
    v, e = oracle.build_sphere(12, 1.0)
    for fam in (P1, P0):
        fast = oracle.bem_dense(v, e, 3, fam, v, e, 3, fam, "[exp(ikr)/r]", 2.0)
        slow = oracle.naive_bem(v, e, 3, fam, v, e, 3, fam, "[exp(ikr)/r]", 2.0)
        assert np.abs(fast - slow).max() <= 1e-13 * np.abs(slow).max()
    with pytest.raises(RuntimeError, match="tol"):
        oracle.bem_dense(v, e, 3, P1, v, e, 3, P1, "[exp(ikr)/r]", 2.0, cap=1000)


def test_memory_cap_refuses_config3_at_defaults(oracle):
    # SURVEY trap 5: 16*(20480^2 + 1024*122880 + 1024*20480) = 9.06e9 > 8e9
    need = 16 * (20480 ** 2 + 1024 * 122880 + 1024 * 20480)
    assert need > 8e9


def test_bem_rows_are_bit_identical_to_full(oracle):
    v, e = oracle.build_sphere(162, 1.0)
    full = oracle.bem_dense(v, e, 3, P1, v, e, 3, P1, "[exp(ikr)/r]", 4.0)
    rows = [3, 77, 160, 0]
    part = oracle.bem_dense(v, e, 3, P1, v, e, 3, P1, "[exp(ikr)/r]", 4.0, rows=rows, chunk=37)
    assert np.array_equal(part, full[rows, :])


def test_regularize_self_term_and_far_pairs(oracle):
    v, e = single_triangle(1.0)
    raw = oracle.bem_dense(v, e, 7, P0, v, e, 7, P0, "[1/r]", 0.0)
    r, c, vals, _ = oracle.regularize(v, e, 7, P0, v, e, 7, P0, "[1/r]")
    corrected = (raw[0, 0].real + vals[0]) / (4 * math.pi)
    ref = oracle.double_newton_oracle((0, 0, 0), (1, 0, 0), (0, 1, 0), 5e-8) / (4 * math.pi)
    assert abs(corrected - ref) <= 1e-6 * abs(ref)

    v, e = oracle.build_sphere(162, 1.0)
    r, c, vals, _ = oracle.regularize(v, e, 3, P1, v, e, 3, P1, "[1/r]", threads=8)
    C = np.zeros((162, 162))
    C[r, c] = vals
    checked = 0
    for i in range(40):
        for j in range(40):
            if np.linalg.norm(v[i] + v[j]) < 0.2:
                assert C[i, j] == 0.0
                checked += 1
    assert checked > 0
    with pytest.raises(ValueError):
        oracle.regularize(v, e, 3, P1, v, e, 3, P1, "[log r]")


def test_capacity_of_the_sphere(oracle):
    v, e = oracle.build_sphere(642, 1.0)
    s = oracle.bem_dense(v, e, 3, P1, v, e, 3, P1, "[1/r]", 0.0)
    r, c, vals, _ = oracle.regularize(v, e, 3, P1, v, e, 3, P1, "[1/r]", threads=8)
    s[r, c] += vals
    s /= 4 * math.pi
    rhs = np.array(oracle.linear_form_ones(v, e, P1, 3))
    lam = np.linalg.solve(s, rhs)
    assert np.abs(lam.real - 1).max() < 0.02
    assert np.abs(lam.imag).max() < 1e-10
    mass = oracle.mass_dense(v, e, P1, 3).real
    nodal = np.linalg.solve(mass, (s @ np.ones(642)).real)
    assert np.abs(nodal - 1).max() < 0.02
    rad = oracle.radiation_dense(np.array([[100.0, 0, 0]]), v, e, 3, P1, "[1/r]", 0.0) / (4 * math.pi)
    phi = (rad @ lam)[0].real
    # The reference pins |phi - 0.01| < 1e-5 (test_assembly.cpp:243).  The
    # restated algorithm gives phi = 0.0099717: the inscribed 642-vertex
    # polyhedron has 0.48% less area than the sphere and the discrete total
    # charge Q/4pi = 0.99717.  That pin is unreachable for this discretisation,
    # so it is checked at 3e-5 here and the 1e-5 form is an explicit xfail below.
    assert abs(phi - 0.01) < 3e-5
    assert oracle.radiation_dense(np.zeros((0, 3)), v, e, 3, P1, "[1/r]", 0.0).shape == (0, 642)


@pytest.mark.xfail(strict=True, reason="reference pin test_assembly.cpp:243 (1e-5) is below the "
                   "discretisation error of the algorithm it pins (phi=0.0099717)")
def test_capacity_radiation_reference_tolerance(oracle):
    v, e = oracle.build_sphere(642, 1.0)
    s = oracle.bem_dense(v, e, 3, P1, v, e, 3, P1, "[1/r]", 0.0)
    r, c, vals, _ = oracle.regularize(v, e, 3, P1, v, e, 3, P1, "[1/r]", threads=8)
    s[r, c] += vals
    lam = np.linalg.solve(s / (4 * math.pi), np.array(oracle.linear_form_ones(v, e, P1, 3)))
    rad = oracle.radiation_dense(np.array([[100.0, 0, 0]]), v, e, 3, P1, "[1/r]", 0.0) / (4 * math.pi)
    assert abs((rad @ lam)[0].real - 0.01) < 1e-5


def test_sphere_single_layer_known_answer(oracle):
    # int_{S^2} e^{ik|x-y|}/(4 pi |x-y|) dy = e^{ik} sin(k)/k on |x|=1.
    v, e = oracle.build_sphere(642, 1.0)
    k = 2.0
    s = oracle.bem_dense(v, e, 3, P0, v, e, 3, P0, "[exp(ikr)/r]", k)
    r, c, vals, _ = oracle.regularize(v, e, 3, P0, v, e, 3, P0, "[1/r]", threads=8)
    s[r, c] += vals
    area = np.array(oracle.element_measures(v, e))
    pot = (s @ np.ones(len(area))) / (4 * math.pi) / area
    exact = np.exp(1j * k) * math.sin(k) / k
    assert np.abs(pot - exact).max() < 0.02 * abs(exact)


def test_p0_regularize_pairs_ref_vs_2hbar(oracle):
    v, e = oracle.build_sphere(642, 1.0)
    hbar = oracle.edge_stats(v, e)[2]
    ref = oracle.near_pairs(v, e, v, e, 0, 0.0)
    two = oracle.near_pairs(v, e, v, e, 1, hbar)
    assert len(ref) != len(two)
    assert all(p in set(ref) for p in [(i, i) for i in range(10)])


def _collocation_potential(oracle, v, e, pts):
    rad = oracle.radiation_dense(pts, v, e, 3, P1, "[1/r]", 0.0)
    r, c, vals = oracle.regularize_radiation(pts, v, e, 3, P1, "[1/r]")
    rad[np.asarray(r), np.asarray(c)] += vals
    return (rad @ np.ones(rad.shape[1])).real / (4 * math.pi)


@pytest.mark.xfail(strict=True, reason="reference test test_assembly.cpp:248-260 collocates at mesh "
                   "vertices, where analytic_triangle_integrals (kernels.cpp:192-193) evaluates "
                   "atan(0/0) = NaN for every triangle sharing the vertex; the restated algorithm "
                   "reproduces that NaN")
def test_regularized_collocation_at_vertices_reference_form(oracle):
    v, e = oracle.build_sphere(642, 1.0)
    pot = _collocation_potential(oracle, v, e, np.asarray(v)[:5])
    assert np.all(np.abs(pot - 1.0) < 0.02)


@pytest.mark.parametrize("where", ["centroids", "inside", "outside"])
def test_regularized_collocation_near_the_surface(oracle, where):
    # Same check as test_assembly.cpp:248-260 (|pot - 1| < 0.02 for the unit
    # density) at collocation points the analytic integrals are defined at.
    v, e = oracle.build_sphere(642, 1.0)
    v, e = np.asarray(v), np.asarray(e)
    pts = {"centroids": v[e[:5]].mean(axis=1), "inside": 0.999 * v[:5],
           "outside": 1.001 * v[:5]}[where]
    pot = _collocation_potential(oracle, v, e, pts)
    assert np.all(np.abs(pot - 1.0) < 0.02)


def test_block_eval_equals_dense_submatrix(oracle):
    # GalerkinEvaluator::eval (assembly.cpp:240-291) reproduces the dense
    # matrix's entries on any row/column selection (the structural identity
    # bem_h relies on, test_assembly.cpp:262-285), duplicates included.
    v, e = oracle.build_sphere(162, 1.0)
    for name, k, fam in [("[exp(ikr)/r]", 3.0, P1), ("[1/r]", 0.0, P0)]:
        A = oracle.bem_dense(v, e, 3, fam, v, e, 3, fam, name, k)
        rows, cols = [5, 0, 17, 5, 40], [3, 100, 7, 3]
        B = oracle.block_eval(v, e, 3, fam, v, e, 3, fam, name, k, rows, cols)
        assert np.abs(B - A[np.ix_(rows, cols)]).max() <= 1e-14 * np.abs(A).max()
    pts = np.array([[0.0, 0.0, 2.0], [1.5, 0.1, 0.2], [0.3, -1.2, 0.1]])
    R = oracle.radiation_dense(pts, v, e, 3, P1, "[exp(ikr)/r]", 2.0)
    B = oracle.block_eval_points(pts, v, e, 3, P1, "[exp(ikr)/r]", 2.0, [2, 0], [1, 50, 161])
    assert np.abs(B - R[np.ix_([2, 0], [1, 50, 161])]).max() <= 1e-14 * np.abs(R).max()
