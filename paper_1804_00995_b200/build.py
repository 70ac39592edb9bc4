"""Build the sm_100a library and its Python binding in-tree.

Outputs (git-ignored, shipped to the GPU box with the snapshot):
  paper_1804_00995_b200/_build/libgalerk_b200.so   C-ABI (include/galerk_b200.h)
  paper_1804_00995_b200/_build/_galerk<EXT>.so      pybind11 host API
  paper_1804_00995_b200/_build/ptxas.log            -Xptxas -v register/spill report

Usage: python paper_1804_00995_b200/build.py [--force]
"""
import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "_build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = "/usr/bin/g++"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["gk_abi.cu", "gk_assembly.cu", "gk_matvec.cu", "gk_green.cu", "gk_nearfield.cu", "gk_blockeval.cu", "gk_solve.cu",
              "gk_diag.cu"]
CXX_SOURCES = ["gk_plan.cpp", "host/galerk.cpp"]
# tuning experiments only (e.g. GK_NVCC_EXTRA="-DGK_NF_MINB=3"); empty by default
EXTRA = os.environ.get("GK_NVCC_EXTRA", "").split()
HEADERS = ["gk_internal.hpp", "gk_math.cuh", "host/galerk.hpp", "../../include/galerk_b200_diag.h"]


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd, log=None):
    res = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        log.write(" ".join(cmd) + "\n" + res.stdout + res.stderr + "\n")
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd))
    return res


def build(force=False, verbose=False):
    os.makedirs(OUT, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "galerk_b200.h")]
    objs = []
    changed = force
    with open(os.path.join(OUT, "ptxas.log"), "a") as log:
        for src in CU_SOURCES:
            s = os.path.join(CSRC, src)
            o = os.path.join(OUT, os.path.basename(src) + ".o")
            objs.append(o)
            if force or _newer(o, [s] + hdrs):
                changed = True
                # per-source register/spill report of the latest compile (+ the running log)
                with open(o + ".ptxas", "w") as one:
                    res = _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-ccbin", CXX, "-Xcompiler",
                                "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr", *EXTRA, "-c", s, "-o", o], log)
                    one.write(res.stdout + res.stderr)
        for src in CXX_SOURCES:
            s = os.path.join(CSRC, src)
            o = os.path.join(OUT, os.path.basename(src) + ".o")
            objs.append(o)
            if force or _newer(o, [s] + hdrs):
                changed = True
                _run([CXX, "-O3", "-std=c++17", "-fPIC", "-ffp-contract=off", "-Wall", "-Wextra",
                      "-I/usr/local/cuda/include", *EXTRA, "-c", s, "-o", o], log)
    lib = os.path.join(OUT, "libgalerk_b200.so")
    if changed or not os.path.exists(lib):
        _run([NVCC, *ARCH, "-shared", "-ccbin", CXX, "-o", lib, *objs, "-cudart", "static"])
    # python binding
    import pybind11

    ext = sysconfig.get_config_var("EXT_SUFFIX")
    pyso = os.path.join(OUT, "_galerk" + ext)
    pysrc = os.path.join(CSRC, "py", "galerk_py.cpp")
    if force or _newer(pyso, [pysrc, lib] + hdrs):
        _run([CXX, "-O3", "-std=c++17", "-fPIC", "-shared", "-ffp-contract=off",
              "-I" + sysconfig.get_paths()["include"], "-I" + pybind11.get_include(),
              pysrc, "-o", pyso, "-L" + OUT, "-lgalerk_b200", "-Wl,-rpath,$ORIGIN"])
    if verbose:
        print("built", lib, pyso)
    return lib, pyso


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
