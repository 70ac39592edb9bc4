"""Golden fixtures (tests/golden/golden_v1.npz, written by make_golden.py from
the oracle): the oracle must keep reproducing them bit for bit, and the
product's host tables must match the fixture meshes bit for bit."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import make_golden  # noqa: E402

from tests._support import load_oracle, load_product  # noqa: E402


def _golden():
    return np.load(os.path.join(HERE, "golden", "golden_v1.npz"))


def test_oracle_reproduces_the_golden_fixtures_bitwise():
    g = _golden()
    fresh = make_golden.build(load_oracle())
    assert sorted(fresh) == sorted(g.files)
    for key in g.files:
        assert np.array_equal(np.asarray(fresh[key]), g[key]), key


def test_product_meshes_match_the_fixtures():
    g = _golden()
    p = load_product()
    m = p.build_sphere(162, 1.0)
    assert np.array_equal(np.asarray(m.vertices), g["l2_vertices"])
    assert np.array_equal(np.asarray(m.elements), g["l2_elements"])
    m1 = p.perturb_radial(p.build_sphere(42, 1.0), 2, 0.02)
    assert np.array_equal(np.asarray(m1.vertices), g["l1p_vertices"])
    pts, _, _ = p.quadrature(p.make_domain(m, 3))
    assert np.array_equal(np.asarray(pts), g["green_l2_points"])
