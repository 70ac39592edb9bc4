"""GPU parity: batched block evaluation (GalerkinEvaluator::eval, the entry
generator of the H-matrix path, assembly.cpp:225-299) vs the oracle."""
import numpy as np
import pytest

from tests._support import rel_fro, sphere_problem

pytestmark = pytest.mark.gpu
P0, P1 = 0, 1
FAM = {"P0": P0, "P1": P1}


@pytest.mark.parametrize("name,k,fam,gauss", [("[exp(ikr)/r]", 5.0, "P1", 3), ("[1/r]", 0.0, "P0", 3),
                                              ("[exp(ikr)/r]", 2.0, "P0", 7), ("[exp(ikr)/r]", 4.0, "P1", 6)])
def test_eval_matches_oracle(galerk, oracle, name, k, fam, gauss):
    m, dom, sp, _ = sphere_problem(galerk, 642, gauss, fam)
    v, e = np.asarray(m.vertices), np.asarray(m.elements)
    ev = galerk.GalerkinEvaluator(dom, dom, sp, galerk.green_kernel(name, k), sp)
    n = sp.free_count()
    assert ev.rows() == n and ev.cols() == n
    rng = np.random.default_rng(3)
    shapes = [(1, n), (n, 1), (37, 53), (64, 64)]
    for nr, nc in shapes:
        rows = [int(x) for x in rng.integers(0, n, nr)]
        cols = [int(x) for x in rng.integers(0, n, nc)]
        got = ev.eval(rows, cols)
        ref = oracle.block_eval(v, e, gauss, FAM[fam], v, e, gauss, FAM[fam], name, k, rows, cols)
        assert got.shape == (nr, nc)
        assert rel_fro(got, ref) <= 1e-10
        if name == "[1/r]":
            assert np.all(got.imag == 0.0)


def test_eval_batch_and_edge_cases(galerk, oracle):
    m, dom, sp, _ = sphere_problem(galerk, 162, 3, "P1")
    v, e = np.asarray(m.vertices), np.asarray(m.elements)
    kern = galerk.green_kernel("[exp(ikr)/r]", 3.0)
    ev = galerk.GalerkinEvaluator(dom, dom, sp, kern, sp)
    req = [([5, 0, 17, 5], [3, 100, 7]), ([], [1, 2]), ([4], []), (list(range(162)), [9]), ([1], list(range(162)))]
    outs = ev.eval_batch(req)
    for (r, c), got in zip(req, outs):
        assert got.shape == (len(r), len(c))
        if len(r) and len(c):
            ref = oracle.block_eval(v, e, 3, P1, v, e, 3, P1, "[exp(ikr)/r]", 3.0, r, c)
            assert rel_fro(got, ref) <= 1e-10
            assert np.array_equal(got, ev.eval(r, c))  # batching does not change results
    A = galerk.bem_dense(dom, dom, sp, kern, sp)
    assert rel_fro(outs[0], A[np.ix_(req[0][0], req[0][1])]) <= 1e-10
    with pytest.raises(ValueError):
        ev.eval([162], [0])
    with pytest.raises(ValueError):
        ev.eval([0], [-1])


def test_points_evaluator_matches_radiation(galerk, oracle):
    m, dom, sp, _ = sphere_problem(galerk, 642, 3, "P1")
    v, e = np.asarray(m.vertices), np.asarray(m.elements)
    rng = np.random.default_rng(5)
    pts = rng.normal(size=(200, 3)) * 2.0
    kern = galerk.green_kernel("[exp(ikr)/r]", 4.0)
    ev = galerk.GalerkinEvaluator.points(pts, dom, kern, sp)
    assert ev.rows() == 200
    rows, cols = list(range(0, 200, 3)), list(range(0, 642, 5))
    got = ev.eval(rows, cols)
    ref = oracle.block_eval_points(pts, v, e, 3, P1, "[exp(ikr)/r]", 4.0, rows, cols)
    assert rel_fro(got, ref) <= 1e-10
    R = galerk.radiation_dense(pts, dom, kern, sp)
    assert rel_fro(got, R[np.ix_(rows, cols)]) <= 1e-10


def _aca(ev, rows, cols, tol):
    """Partial-pivot ACA over evaluator panels (the algorithm of hmatrix.cpp aca):
    every row / column panel is one device round trip."""
    m, n = len(rows), len(cols)
    U, V, used = [], [], set()
    i, norm2 = 0, 0.0
    for _ in range(min(m, n)):
        used.add(i)
        row = ev.eval([rows[i]], cols)[0].copy()
        for u, w in zip(U, V):
            row -= u[i] * w
        j = int(np.argmax(np.abs(row)))
        if abs(row[j]) == 0.0:
            break
        w = row / row[j]
        col = ev.eval(rows, [cols[j]])[:, 0].copy()
        for u, x in zip(U, V):
            col -= x[j] * u
        for u, x in zip(U, V):
            norm2 += 2.0 * np.real(np.vdot(u, col) * np.vdot(x, w))
        nu, nw = np.linalg.norm(col), np.linalg.norm(w)
        norm2 += (nu * nw) ** 2
        U.append(col)
        V.append(w)
        if nu * nw <= tol * np.sqrt(norm2):
            break
        cand = np.abs(col)
        cand[list(used)] = -1.0
        i = int(np.argmax(cand))
    return np.array(U).T, np.array(V).T


def test_aca_on_admissible_block(galerk):
    """ACA (compressed path) driven by device panels reproduces a far block."""
    m, dom, sp, _ = sphere_problem(galerk, 2562, 3, "P1")
    v = np.asarray(m.vertices)
    kern = galerk.green_kernel("[exp(ikr)/r]", 5.0)
    ev = galerk.GalerkinEvaluator(dom, dom, sp, kern, sp)
    rows = [int(i) for i in np.where(v[:, 2] > 0.8)[0]]
    cols = [int(i) for i in np.where(v[:, 2] < -0.8)[0]]
    U, V = _aca(ev, rows, cols, 1e-6)
    B = ev.eval(rows, cols)
    assert U.shape[1] < min(len(rows), len(cols)) // 4
    assert np.linalg.norm(B - U @ V.T) <= 1e-5 * np.linalg.norm(B)
