"""galerk_b200 — B200-native (sm_100a) dense Galerkin BEM hot path.

A drop-in for the dense assembly path of the `galerk` reference
(Gypsilab-in-C++): ``bem_dense`` / ``radiation_dense`` / ``regularize`` and the
stored / matrix-free Green-kernel matvecs, computed by hand-written CUDA
kernels behind the C-ABI in ``include/galerk_b200.h``.

There is no CPU fallback: importing fails loudly if the in-tree extension
(``_build/_galerk*.so``, built by ``python -m paper_1804_00995_b200.build``) is
missing, and every compute call fails without a CUDA device.
"""
import glob
import importlib.util
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
_BUILD = os.path.join(_HERE, "_build")


def _load():
    cands = glob.glob(os.path.join(_BUILD, "_galerk*.so"))
    if not cands:
        raise ImportError(
            "galerk_b200 native extension not built (expected paper_1804_00995_b200/_build/_galerk*.so); "
            "run `python paper_1804_00995_b200/build.py` — there is no CPU fallback")
    spec = importlib.util.spec_from_file_location("_galerk", cands[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


_native = _load()

Mesh = _native.Mesh
EdgeStats = _native.EdgeStats
build_sphere = _native.build_sphere
edge_stats = _native.edge_stats
perturb_radial = _native.perturb_radial
Domain = _native.Domain
make_domain = _native.make_domain
supported_rules = _native.supported_rules
reference_rule = _native.reference_rule
quadrature = _native.quadrature
Family = _native.Family
FemSpace = _native.FemSpace
make_fem = _native.make_fem
Kernel = _native.Kernel
green_kernel = _native.green_kernel
BemOptions = _native.BemOptions
bem_dense = _native.bem_dense
radiation_dense = _native.radiation_dense
regularize = _native.regularize
regularize_radiation = _native.regularize_radiation
AssemblyPlan = _native.AssemblyPlan
GreenPlan = _native.GreenPlan
NearField = _native.NearField
GalerkinEvaluator = _native.GalerkinEvaluator
NEAR_REF = _native.NEAR_REF
NEAR_2HBAR = _native.NEAR_2HBAR
matvec = _native.matvec
matvec_launches = _native.matvec_launches
matvec_multi = _native.matvec_multi
matvec_multi_launches = _native.matvec_multi_launches
evaluate_blocks = _native.evaluate_blocks
lu_factor = _native.lu_factor
lu_solve = _native.lu_solve
gmres = _native.gmres
side_tables = _native.side_tables
uniform01 = _native.uniform01
normal = _native.normal
complex_normal = _native.complex_normal
bem_dense_into = _native.bem_dense_into
diag_fp64_peak = _native.diag_fp64_peak
diag_fp64_sustained = _native.diag_fp64_sustained
plan_info_dry = _native.plan_info_dry
plan_info_dry_rows = _native.plan_info_dry_rows
location_ids = _native.location_ids
diag_probe_pairs = _native.diag_probe_pairs
diag_probe_analytic = _native.diag_probe_analytic
diag_math = _native.diag_math
last_error = _native.last_error
version = _native.version
FP64 = _native.FP64
FP32 = _native.FP32

LIBRARY_PATH = os.path.join(_BUILD, "libgalerk_b200.so")

__all__ = [n for n in dir() if not n.startswith("_")]
