"""Test helpers: load (building if needed) the oracle and the product."""
import glob
import importlib
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_oracle():
    """The CPU oracle (test infrastructure only)."""
    build = os.path.join(ROOT, "oracle", "_build")
    if not glob.glob(os.path.join(build, "_oracle*.so")):
        subprocess.check_call(["make", "-C", os.path.join(ROOT, "oracle")])
    if build not in sys.path:
        sys.path.insert(0, build)
    return importlib.import_module("_oracle")


def load_product():
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    import paper_1804_00995_b200 as g

    return g


def rel_fro(a, b):
    """Relative Frobenius error ||a-b||_F / ||b||_F."""
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def colmajor_from_torch(t, rows, cols, lda):
    """Device buffer (complex128, col-major, leading dim lda) -> numpy (rows, cols)."""
    a = t.detach().cpu().numpy().reshape(cols, lda)
    return np.ascontiguousarray(a[:, :rows].T)


def sphere_problem(g, n_target, gauss, family, perturb_seed=None):
    """Product-side mesh/domain/space; returns (mesh, dom, space, hbar)."""
    mesh = g.build_sphere(n_target, 1.0)
    if perturb_seed is not None:
        mesh = g.perturb_radial(mesh, perturb_seed, 0.02)
    dom = g.make_domain(mesh, gauss)
    space = g.make_fem(mesh, family)
    hbar = g.edge_stats(mesh).mean_len
    return mesh, dom, space, hbar


def load_ref():
    """The reference's own mesh/quadrature/kernel sources compiled against the
    Eigen-API shim (oracle/Makefile `ref`, test infrastructure), or None where
    neither the built module nor /root/reference is available."""
    out = os.path.join(ROOT, "oracle", "_ref")
    if not glob.glob(os.path.join(out, "_ref*.so")):
        if not os.path.isdir("/root/reference/proj/src"):
            return None
        subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"])
    if out not in sys.path:
        sys.path.insert(0, out)
    return importlib.import_module("_ref")
