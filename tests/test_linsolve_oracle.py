"""Pins the numpy GMRES restatement (oracle/linsolve_oracle.py) to the
reference's own linsolve tests (test_linsolve.cpp:10-28) — CPU only."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import linsolve_oracle  # noqa: E402


def test_gmres_trivial_systems():
    n = 10
    b = np.linspace(1.0, 10.0, n)
    x, info = linsolve_oracle.gmres(lambda v: v, b, 1e-12)
    assert info["converged"] and info["iterations"] <= 1
    assert np.linalg.norm(x - b) < 1e-12
    d = np.arange(1, n + 1, dtype=float)
    x2, info2 = linsolve_oracle.gmres(lambda v: v * d, np.ones(n), 1e-12)
    assert info2["converged"]
    assert np.allclose(x2.real, 1.0 / d, rtol=1e-10, atol=0)


def test_gmres_dense_system_history_monotone():
    rng = np.random.default_rng(0)
    n = 120
    A = np.eye(n) * 4 + rng.normal(size=(n, n)) / np.sqrt(n) + 1j * rng.normal(size=(n, n)) / np.sqrt(n)
    b = rng.normal(size=n) + 1j * rng.normal(size=n)
    x, info = linsolve_oracle.gmres(lambda v: A @ v, b, 1e-10, restart=20, maxit=500)
    assert info["converged"]
    assert np.linalg.norm(A @ x - b) / np.linalg.norm(b) <= 1e-10
    h = info["history"]
    assert all(h[i] <= h[i - 1] * (1 + 1e-10) + 1e-14 for i in range(1, len(h)))  # test_linsolve.cpp:46-48


def test_gmres_rejects_bad_tolerance():
    with pytest.raises(ValueError, match="tol must be positive"):
        linsolve_oracle.gmres(lambda v: v, np.ones(3), 0.0)
