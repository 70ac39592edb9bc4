#!/usr/bin/env python
"""bench.py — driver-contract benchmark for the B200 dense BEM hot path.

Default workload (BASELINE.json configs[3], "cfg4", the largest configuration
that fits one GPU): unit-sphere icosphere L6 (40962 vertices, 81920
triangles), P0, 3-point (edge-midpoint) rule, Helmholtz single layer with
k = 2 pi / (10 hbar).  One step = dense assembly of the 81920 x 81920
complex128 matrix (107 GB, resident in HBM; K1+K2) followed by 10 stored
matvecs y = A x (K4) with seeded complex N(0,1) vectors (seed 3).  The ten
vectors are independent, so the step multiplies them in one pass over A
(gk_matvec_multi, Y = A X; --matvec single: one gk_matvec per vector, ten
passes).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--config 1|2|3|4|5] [--extras 2,3,5|none]

Metric: reference-equivalent quadrature-pair kernel evaluations per second
(M_x * M_y per step / step time).  `roofline` is the assembly kernel against
the FP64 pipe (sustained DFMA peak measured in the same run); `roofline_matvec`
the single-vector stored matvec against HBM; `roofline_matvec_multi` the
step's one-pass multiply of all vectors (FP64 or HBM, whichever binds).  With the default config the cfg 2 / cfg 3 /
cfg 5 lines (smaller workloads, BASELINE configs[1], [2], [4]) are measured
first and nested under "other_configs".

--impl reference: the reference's CPU path (the oracle restatement of
bem_product / regularize / zgemv / the matrix-free loop, oracle/; the
reference itself cannot be built here) on all host cores, on
the same config, metric and unit; it imports nothing from the product.
Multi-GPU: replicas only — every rank runs the full step; value
is the whole-job aggregate over ranks with the max-over-ranks device time.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0  # B200_PROFILING.md fallback if MEASURED_PEAKS.json is absent
# FP64 work per unique location pair (DESIGN.md §4 "F_pair"), frozen from ncu
# counters (profiles/r01_fpair_probe.txt): the canonical probe —
# the reference formula kernels.cpp:94-114 with libdevice sqrt/sin/cos/division
# plus one complex x real accumulate — 43 DFMA + 13 DMUL + 7 DADD = 106
# flops/pair (DFMA = 2 flops); Laplace ("[1/r]") 23 flops.
F_PAIR_PROBE_FLOPS = {True: 106.0, False: 23.0}
# the production pair loop (SASS count incl. the y-side accumulation), for
# the executed-work fraction: P1 cfg 2 23 DFMA + 7 DMUL + 4 DADD = 57 flops/pair
F_PAIR_PROD_FLOPS = {True: 57.0, False: 19.0}
# F_analytic: FP64 flops of one reference analytic_triangle_integrals
# call (kernels.cpp:151-207 with libdevice log/atan/sqrt/division), frozen by ncu
# on the cfg-3 call mix (scripts/fanalytic_probe.py, profiles/r02_fanalytic_probe.txt):
# 395.8 DFMA + 135.1 DMUL + 108.0 DADD per call = 1034.7 flops.
F_ANALYTIC_FLOPS = 1034.7
METRIC = "quadrature-pair kernel evals/s (reference-equivalent M_x*M_y per step, fp64)"
METRIC_GREEN = "matrix-free Green matvec pair evals/s (reference-equivalent M^2 per matvec, fp64)"

SPECS = {
    1: dict(n=642, gauss=3, fam="P1", helm=False, perturb=None, seed=0, real_x=True, nmv=1),
    2: dict(n=10242, gauss=3, fam="P1", helm=True, perturb=None, seed=1, real_x=False, nmv=1),
    3: dict(n=10242, gauss=6, fam="P0", helm=True, perturb=2, seed=1, real_x=False, nmv=1),
    4: dict(n=40962, gauss=3, fam="P0", helm=True, perturb=None, seed=3, real_x=False, nmv=10),
    5: dict(n=163842, gauss=3, fam="points", helm=True, perturb=None, seed=4, real_x=False, nmv=1),
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["b200", "reference"], default="b200")
    p.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5])
    p.add_argument("--extras", default=None,
                   help="comma list of extra configs measured first (default: 2,3,5 with --config 4 at N=1)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--cpu-chunks", type=int, default=8, help="1024-point x chunks of the 1-thread CPU baseline")
    p.add_argument("--matvec", choices=["multi", "single"], default="multi",
                   help="the step's stored matvecs: one pass over A for all vectors (gk_matvec_multi) or one "
                        "gk_matvec per vector")
    return p.parse_args()


# ---------------------------------------------------------------------------------
def workload_name(cfg, nv, ne):
    return {
        1: f"cfg1: Laplace single layer, P1, 3-pt, icosphere L3 ({nv} v/{ne} t), 642^2 real-valued complex128 + matvec",
        2: f"cfg2: Helmholtz single layer, P1, 3-pt, icosphere L5 ({nv} v/{ne} t), 10242^2 complex128 + matvec",
        3: f"cfg3: Helmholtz single layer, P0, 6-pt, perturbed L5 ({ne} t), 20480^2 complex128 incl. near-field "
           f"correction + matvec",
        4: f"cfg4: Helmholtz single layer, P0, 3-pt, icosphere L6 ({ne} t), 81920^2 complex128 (107 GB in HBM) "
           f"+ 10 stored matvecs",
        5: f"cfg5: matrix-free Helmholtz Green matvec, 983040 points = 3-pt Gauss nodes of icosphere L7 ({ne} t), "
           f"self-interaction masked",
    }[cfg]


def config_dict(cfg, nv, ne, N, M, k, hbar):
    """The `config` object — identical on both arms (built from their own, bitwise
    identical, mesh statistics)."""
    s = SPECS[cfg]
    d = {"workload": workload_name(cfg, nv, ne), "N": int(N), "M": int(M), "k": float(k), "hbar": float(hbar),
         "space": s["fam"], "rule_points": s["gauss"], "matvecs_per_step": s["nmv"] if cfg != 5 else 0}
    if cfg == 5:
        d["l2"] = "matrix-free: sources (15.7 MB fp64) re-streamed from L2 per tile"
    else:
        d["l2"] = "inputs larger than L2 for cfg 2-4: A = %.2f GB written and read every step (no flush needed)" % (
            16.0 * N * N / 1e9)
    return d


# ---------------------------------------------------------------------------------
class ClockSampler:
    """SM clock + throttle reasons sampled during the timed region (NVML, 5 ms
    period; falls back to nvidia-smi at 200 ms)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, power_w, reasons_mask)
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception:
            self._nv = None

    def _sample(self):
        if self._nv is not None:
            nv, h = self._nv, self._h
            return (float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                    float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)),
                    nv.nvmlDeviceGetPowerUsage(h) / 1000.0,
                    int(nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
        out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                              "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
        c = [x.strip() for x in out.stdout.strip().split(",")]
        return float(c[0]), float(c[1]), float(c[2]), int(c[3], 16)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.rows.append(self._sample())
            except Exception:
                pass
            self._stop.wait(0.005 if self._nv is not None else 0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)
        try:  # one sample at the end of the region as well
            self.rows.append(self._sample())
        except Exception:
            pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"], "samples": 0}
        reasons = sorted({n for r in self.rows for n, bit in self.REASONS.items() if r[3] & bit})
        return {"sm_mhz": float(np.median([r[0] for r in self.rows])), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": reasons, "samples": len(self.rows), "power_w_max": max(r[2] for r in self.rows),
                "source": "nvml" if self._nv is not None else "nvidia-smi"}


def max_over_ranks(ms, dist, device):
    """Device-timed milliseconds -> max over all ranks (replicas finish when the slowest does)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(ms)
    import torch

    t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_value(units_per_rank, world, ms_step):
    """Whole-job throughput: units of all ranks / the max-over-ranks step time."""
    return world * units_per_rank / (ms_step * 1e-3)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def profile_summary(cfg):
    """The committed ncu capture of the dominant kernel (profiles/ncu_summary.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f).get(f"cfg{cfg}", {})
    except Exception:
        return {}


# ---------------------------------------------------------------------------------
# CPU side (oracle = test infrastructure: only the cpu_baseline leg and the
# reference arm run it).  Chunks follow SURVEY §8(d): S uniformly spaced
# 1024-point chunks of the x quadrature points (the reference's
# BemOptions::chunk, assembly.cpp:212-220); the oracle computes the complete
# rows of the test dofs those points support (bitwise the full computation's
# rows) and the time extrapolates linearly in the x points processed.
def load_oracle():
    from tests._support import load_oracle as _lo

    return _lo()


def oracle_problem(o, cfg):
    """Mesh statistics and side tables from the oracle alone (reference arm: no
    product code is imported)."""
    s = SPECS[cfg]
    v, e = o.build_sphere(s["n"], 1.0)
    if s["perturb"] is not None:
        v, e = o.perturb_radial(v, e, s["perturb"], 0.02)
    v, e = np.asarray(v), np.asarray(e)
    hbar = o.edge_stats(v, e)[2]
    k = 2 * math.pi / (10 * hbar) if s["helm"] else 0.0
    name = "[exp(ikr)/r]" if s["helm"] else "[1/r]"
    fam = {"P1": 1, "P0": 0, "points": 0}[s["fam"]]
    ne, nv = len(e), len(v)
    N = nv if s["fam"] == "P1" else ne
    return dict(v=v, e=e, hbar=hbar, k=k, name=name, fam=fam, ne=ne, nv=nv, N=N, M=ne * s["gauss"], g=s["gauss"])


def chunk_rows(o, P, nchunks, chunk=1024, first=0):
    """Test dofs supported by `nchunks` uniformly spaced 1024-point x chunks."""
    start, dof, _ = o.eval_rows(P["v"], P["e"], P["fam"], P["g"])
    start, dof = np.asarray(start), np.asarray(dof)
    M = P["M"]
    los = np.linspace(0, max(0, M - chunk), max(1, nchunks)).astype(np.int64)
    out = []
    for lo in los[first:]:
        hi = min(M, lo + chunk)
        out.append(sorted(set(dof[start[lo]:start[hi]].tolist())))
    # x points the complete rows touch (what the oracle's row restriction processes)
    pt_of = np.repeat(np.arange(M), np.diff(start))
    npts = [int(len(np.unique(pt_of[np.isin(dof, r)]))) for r in out]
    return out, npts


def complex_normal_np(o, seed, n):
    """n complex N(0,1) values from the SplitMix64 stream `seed` (re then im,
    Box-Muller cos branch first): the product's complex_normal
    (host/galerk.cpp:690-707) drawn from the oracle's stream (numpy libm)."""
    m = 2 * n
    u = np.asarray(o.uniform01_stream(seed, 2 * ((m + 1) // 2)))
    r = np.sqrt(-2.0 * np.log(1.0 - u[0::2]))
    t = 2.0 * np.pi * u[1::2]
    z = np.empty(2 * len(r))
    z[0::2] = r * np.cos(t)
    z[1::2] = r * np.sin(t)
    z = z[:m]
    return z[0::2] + 1j * z[1::2]


def cpu_dense_step(o, P, cfg, rows, npts, threads, xs):
    """Extrapolated seconds of one reference step (assembly [+ regularize] + nmv
    zgemv) from the complete rows of one chunk."""
    s = SPECS[cfg]
    t0 = time.perf_counter()
    Ar = o.bem_dense(P["v"], P["e"], P["g"], P["fam"], P["v"], P["e"], P["g"], P["fam"], P["name"], P["k"],
                     rows=rows, threads=threads, cap=1e15)
    t_asm = time.perf_counter() - t0
    t_reg = 0.0
    if cfg == 3:  # the step includes regularize (assembly.cpp:609-697) of those test elements
        t0 = time.perf_counter()
        o.regularize(P["v"], P["e"], P["g"], 0, P["v"], P["e"], P["g"], 0, "[1/r]", 0, 0.0, list(rows), threads)
        t_reg = time.perf_counter() - t0
    Ar = np.asfortranarray(Ar)
    t0 = time.perf_counter()
    for i in range(s["nmv"]):
        o.matvec(Ar, xs[i], threads)
    t_mv = time.perf_counter() - t0
    nr = len(rows)
    est = t_asm * P["M"] / npts + (t_reg + t_mv) * P["N"] / nr
    return est, dict(t_asm=t_asm, t_reg=t_reg, t_mv=t_mv, rows=nr, npts=npts)


def cpu_green_step(o, P, threads, ids, eps, q):
    pts, _, _ = o.quadrature(P["v"], P["e"], P["g"])
    pts = np.asarray(pts)
    t0 = time.perf_counter()
    o.green_matvec(P["name"], P["k"], pts, pts, q, eps, list(ids), threads)
    t = time.perf_counter() - t0
    return t * P["M"] / len(ids), t


def cpu_baseline(o, cfg, nchunks, threads=1):
    """The reference's CPU path on `nchunks` chunks, `threads` threads (1 = the
    reference's own concurrency), extrapolated to a full step."""
    P = oracle_problem(o, cfg)
    s = SPECS[cfg]
    if cfg == 5:
        pts, w, _ = o.quadrature(P["v"], P["e"], P["g"])
        pts, w = np.asarray(pts), np.asarray(w)
        q = w * complex_normal_np(o, s["seed"], len(w))
        lo, hi = pts.min(axis=0), pts.max(axis=0)
        eps = 1e-12 * float(np.linalg.norm(hi - lo))  # singular_guard_radius (kernels.cpp:14-19)
        M = P["M"]
        ids = np.concatenate([np.arange(b, b + 16) for b in np.linspace(0, M - 16, max(1, nchunks)).astype(np.int64)])
        est, t = cpu_green_step(o, P, threads, ids, eps, q)
        return {"value": P["M"] ** 2 / est, "unit": "pairs/s", "cores": threads, "kind": "port",
                "sample": f"oracle matrix-free Green matvec (evaluate_blocks mask=true x weighted charges), "
                          f"{len(ids)} targets in {nchunks} uniformly spaced blocks x {M} sources in {t:.1f} s, "
                          f"{threads} thread(s); extrapolated x{M / len(ids):.0f}"}
    xs = [complex_normal_np(o, s["seed"], P["N"] * s["nmv"])[i * P["N"]:(i + 1) * P["N"]] for i in range(s["nmv"])]
    chunks, npts = chunk_rows(o, P, nchunks)
    ests, det = [], []
    for r, n in zip(chunks, npts):
        e, d = cpu_dense_step(o, P, cfg, r, n, threads, xs)
        ests.append(e)
        det.append(d)
    est = float(np.sum([d["t_asm"] for d in det]) * P["M"] / np.sum(npts)
                + np.sum([d["t_reg"] + d["t_mv"] for d in det]) * P["N"] / np.sum([d["rows"] for d in det]))
    tot = sum(d["t_asm"] + d["t_reg"] + d["t_mv"] for d in det)
    return {"value": P["M"] ** 2 / est, "unit": "pairs/s", "cores": threads, "kind": "port",
            "step_s_extrapolated": est,
            "sample": f"oracle bem_product restatement (+ regularize for cfg 3) + {s['nmv']} zgemv on the complete "
                      f"rows of {len(chunks)} uniformly spaced 1024-point x chunks ({sum(d['rows'] for d in det)} rows, "
                      f"{sum(npts)} x points x {P['M']} y points) in {tot:.1f} s, {threads} thread(s); "
                      f"extrapolated linearly in x points (assembly) and rows (matvec)"}


# ---------------------------------------------------------------------------------
def product_problem(g, cfg):
    """Mesh/space/kernel of a BASELINE config through the product's host API."""
    s = SPECS[cfg]
    mesh = g.build_sphere(s["n"], 1.0)
    if s["perturb"] is not None:
        mesh = g.perturb_radial(mesh, s["perturb"], 0.02)
    hbar = g.edge_stats(mesh).mean_len
    k = 2 * math.pi / (10 * hbar) if s["helm"] else 0.0
    name = "[exp(ikr)/r]" if s["helm"] else "[1/r]"
    dom = g.make_domain(mesh, s["gauss"])
    space = g.make_fem(mesh, s["fam"]) if s["fam"] != "points" else None
    return dict(mesh=mesh, dom=dom, space=space, kern=g.green_kernel(name, k), k=k, hbar=hbar, name=name,
                nv=mesh.vertex_count(), ne=mesh.element_count())


def fp64_peaks(g, torch, dev, stream, seconds=2.0):
    """Burst (one short DFMA launch) and sustained (DFMA + 0.125 B/flop of HBM
    stores, back to back for `seconds`) FP64 peaks, measured now."""
    burst = g.diag_fp64_peak(20000, stream.cuda_stream) / 1e3
    scratch = torch.empty(4 << 30, dtype=torch.uint8, device=dev)
    with ClockSampler(dev.index or 0) as clk:
        gf, ms = g.diag_fp64_sustained(seconds, scratch.data_ptr(), scratch.numel(), stream.cuda_stream)
    del scratch
    torch.cuda.empty_cache()
    return burst, gf / 1e3, clk.summary(), ms


def run_dense(args, g, torch, dev, rank, world, dist, cfg, steps, warmup, peaks_fp64, with_cpu, with_e2e):
    s = SPECS[cfg]
    pp = product_problem(g, cfg)
    opts = g.BemOptions()
    opts.memory_cap_bytes = 10 ** 15  # the reference's 8e9 cap refuses cfg 3/4 (SURVEY trap 5)
    space, dom, kern = pp["space"], pp["dom"], pp["kern"]
    plan = g.AssemblyPlan(dom, dom, space, kern, space, opts)
    info = plan.info()
    n = info["rows"]
    nmv = s["nmv"]
    A = torch.empty(n * n, dtype=torch.complex128, device=dev)
    xs = g.normal(s["seed"], n) if s["real_x"] else g.complex_normal(s["seed"], nmv * n)
    X = torch.tensor(np.asarray(xs, dtype=np.complex128).reshape(nmv, n), device=dev)
    y = torch.empty(n, dtype=torch.complex128, device=dev)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    nf = g.NearField(dom, dom, space, "[1/r]", space) if cfg == 3 else None
    multi = args.matvec == "multi" and nmv > 1
    Y = torch.empty((nmv, n), dtype=torch.complex128, device=dev)
    mv_launches = g.matvec_multi_launches(n, n, nmv) if multi else nmv * g.matvec_launches(n, n)
    launches_per_step = plan.launches() + mv_launches + (3 if nf else 0)

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        plan.assemble(A.data_ptr(), n, sp)
        if ev:
            ev[3].record(stream)
        if nf:
            nf.compute(sp)
            nf.apply(A.data_ptr(), n, sp)
        if ev:
            ev[1].record(stream)
        if multi:  # the nmv independent vectors in one pass over A
            g.matvec_multi(A.data_ptr(), n, n, n, X.data_ptr(), n, Y.data_ptr(), n, nmv, sp)
        else:
            for i in range(nmv):
                g.matvec(A.data_ptr(), n, n, n, X[i].data_ptr(), Y[i].data_ptr(), sp)
        if ev:
            ev[2].record(stream)

    for _ in range(max(3, warmup)):
        step()
    torch.cuda.synchronize(dev)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(dev.index or 0) as clk:
        t0.record(stream)
        for i in range(steps):
            step(evs[i])
        t1.record(stream)
        torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    total_ms = max_over_ranks(t0.elapsed_time(t1), dist, dev)
    asm_ms = float(np.mean([e[0].elapsed_time(e[3]) for e in evs]))
    nf_ms = float(np.mean([e[3].elapsed_time(e[1]) for e in evs])) if nf else None
    mvs_ms = float(np.mean([e[1].elapsed_time(e[2]) for e in evs]))  # all of the step's matvecs
    ms_step = total_ms / steps
    # the single-vector stored matvec (K4, HBM-bound) timed on its own
    m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.matvec(A.data_ptr(), n, n, n, X[0].data_ptr(), y.data_ptr(), sp)
    m0.record(stream)
    for _ in range(5):
        g.matvec(A.data_ptr(), n, n, n, X[0].data_ptr(), y.data_ptr(), sp)
    m1.record(stream)
    torch.cuda.synchronize(dev)
    mv_ms = m0.elapsed_time(m1) / 5
    pairs_ref = info["pairs_reference"]
    value = aggregate_value(pairs_ref, world, ms_step)
    # the assembly alone, back to back, under its own clock sampler: the SM
    # clock the kernel itself runs at (the step's median also covers the
    # matvecs; a power-capped box clocks FP64 + store-heavy work lower than
    # the DFMA microbenchmark)
    asm_alone = None
    if rank == 0:
        q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        with ClockSampler(dev.index or 0) as aclk:
            q0.record(stream)
            for _ in range(reps):
                plan.assemble(A.data_ptr(), n, sp)
            q1.record(stream)
            torch.cuda.synchronize(dev)
        asm_alone = {"ms": q0.elapsed_time(q1) / reps, "clocks": aclk.summary()}
    nf_2h = None
    if nf and rank == 0:
        # BASELINE words cfg 3's near field as "pairs closer than 2 hbar"; the
        # reference's rule (used in the step) is 3 max circumradius (SURVEY trap 3).
        nf2 = g.NearField(dom, dom, space, "[1/r]", space, g.NEAR_2HBAR, pp["hbar"])
        nf2.compute(sp)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        nf2.compute(sp)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        nf_2h = {"ms": e0.elapsed_time(e1), "pairs": nf2.info()[0], "analytic_calls": nf2.stats()[0]}
        del nf2
    out = None
    if rank == 0:
        peaks = measured_peaks()
        hbm = peaks.get("hbm_gbs", HBM_FALLBACK_GBS)
        helm = pp["k"] != 0.0
        burst, sustained, sus_clk, sus_ms = peaks_fp64
        achieved = info["pairs_unique"] * F_PAIR_PROBE_FLOPS[helm] / (asm_ms * 1e-3) / 1e12
        exec_prod = info["pairs_evaluated"] * F_PAIR_PROD_FLOPS[helm] / (asm_ms * 1e-3) / 1e12
        mv_bytes = 16.0 * n * n + 32.0 * n
        prof = profile_summary(cfg)
        out = {
            "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": steps, "warmup": warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64 (complex128)",
            "data": "synthetic (seeded icosphere mesh per BASELINE config, SplitMix64/Box-Muller vectors)",
            "config": config_dict(cfg, pp["nv"], pp["ne"], n, math.isqrt(pairs_ref), pp["k"], pp["hbar"])
            | {"parallelism": f"replicas x{world}"},
            "entries_per_s": world * n * n / (ms_step * 1e-3),
            "assembly_ms": asm_ms, "nearfield_ms": nf_ms,
            "nearfield": (dict(zip(("pairs", "entries"), nf.info())) | {"analytic_calls": nf.stats()[0], "rule": "ref"})
            if nf else None,
            "nearfield_2hbar": nf_2h,
            "nearfield_roofline": nearfield_roofline(nf, nf_ms, peaks_fp64) if nf else None,
            "matvec_ms": mv_ms, "matvec_gbs": mv_bytes / (mv_ms * 1e-3) / 1e9,
            "matvecs_step_ms": mvs_ms, "matvec_mode": "multi (gk_matvec_multi: %d vectors, one pass over A)" % nmv
            if multi else "single (one gk_matvec per vector)",
            "unique_pairs_per_s": info["pairs_unique"] / (asm_ms * 1e-3),
            "pairs_evaluated_per_unique": info["pairs_evaluated"] / info["pairs_unique"],
            "plan": {k_: info[k_] for k_ in ("tiles", "x_halo", "y_halo", "natural_order", "device_bytes")},
            "roofline": {"bound": "fp64", "kernel": "k_assemble (K1+K2)", "achieved": achieved, "peak": sustained,
                         "unit": "TFLOP/s", "frac": achieved / sustained,
                         "traffic": prof.get("k_assemble_dram_bytes_per_launch"),
                         "algorithmic_write_bytes": 16.0 * n * n,
                         "peak_source": "sustained FP64 peak measured in this run: DFMA chains + 0.125 B/flop HBM "
                                        "stores, back to back for %.1f s (gk_diag_fp64_sustained; MEASURED_PEAKS.json "
                                        "has no FP64 figure)" % (sus_ms / 1e3),
                         "peak_clocks": sus_clk,
                         "peak_burst": burst, "frac_of_burst": achieved / burst,
                         "work": "pairs_unique (twins merged, symmetric half) x %.0f flops/pair = canonical libdevice "
                                 "probe F_pair (SURVEY 8d)" % F_PAIR_PROBE_FLOPS[helm],
                         "frac_executed_pairs_production_formula": exec_prod / sustained,
                         "assembly_alone": asm_alone,
                         "peak_at_kernel_clock": burst * kernel_clock_ratio(asm_alone, sus_clk),
                         "frac_at_kernel_clock": achieved / (burst * kernel_clock_ratio(asm_alone, sus_clk)),
                         "ncu_fp64_pipe_pct": prof.get("fp64_pipe_pct"),
                         "ncu_sfu_xu_pipe_pct": prof.get("xu_pipe_pct")},
            "roofline_matvec": {"bound": "hbm", "kernel": "k_matvec_partial + k_matvec_reduce (K4)",
                                "achieved": mv_bytes / (mv_ms * 1e-3) / 1e9, "peak": hbm,
                                "unit": "GB/s", "frac": mv_bytes / (mv_ms * 1e-3) / 1e9 / hbm,
                                "traffic": prof.get("k_matvec_dram_bytes_per_call"),
                                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback"},
            "roofline_matvec_multi": (matvec_multi_roofline(n, nmv, mvs_ms, hbm, peaks_fp64)
                                      | {"traffic": prof.get("k_matvec_multi_dram_bytes_per_call"),
                                         "ncu_fp64_pipe_pct": prof.get("k_matvec_multi_fp64_pipe_pct")})
            if multi else None,
            "step_share": {"assembly": asm_ms / ms_step, "nearfield": (nf_ms or 0.0) / ms_step,
                           "matvecs": mvs_ms / ms_step},
            "clocks": clk.summary(),
            "gpu_launches": launches_per_step * steps,
        }
    if with_e2e and rank == 0:
        del A  # the e2e leg allocates its own device matrix
        torch.cuda.empty_cache()
        out["e2e"] = e2e_dense(g, torch, dev, cfg, pp, opts, n, nmv, xs, pairs_ref, steps, warmup, multi)
    if with_cpu and rank == 0 and world == 1:
        R = load_ref_module() if cfg in (1, 2, 4) else None
        if R is not None:  # the reference's own code, one thread, four slices of the mesh (~10-20 s)
            r = reference_arm_compiled(args, R, cfg, threads=1, steps=4, warmup=0)
            out["cpu_baseline"] = {"value": r["value"], "unit": "pairs/s", "cores": 1, "kind": "reference",
                                   "sample": r["sample"]}
        else:
            out["cpu_baseline"] = cpu_baseline(load_oracle(), cfg, args.cpu_chunks if cfg == 4 else 2, threads=1)
    return out


def kernel_clock_ratio(alone, ref_clk):
    """SM clock the assembly ran at (median, sampled while it ran alone) over
    the maximum SM clock the burst DFMA peak is quoted at."""
    try:
        f = alone["clocks"]["sm_mhz"]
        fmax = alone["clocks"]["sm_max_mhz"] or ref_clk.get("sm_max_mhz") or 1965.0
        return min(1.0, float(f) / float(fmax)) if f else 1.0
    except Exception:
        return 1.0


def matvec_multi_roofline(n, nmv, ms, hbm, peaks_fp64):
    """Y = A X over nmv vectors in one pass: 16 N^2 bytes of A (+ X, Y) against
    HBM, and 8 flops per complex multiply-add per vector (4 DFMA) against the
    FP64 pipe; the bound is the larger fraction."""
    t = ms * 1e-3
    gbs = (16.0 * n * n + 32.0 * n * nmv) / t / 1e9
    tfs = 8.0 * n * n * nmv / t / 1e12
    sustained = peaks_fp64[1]
    fh, ff = gbs / hbm, tfs / sustained
    return {"bound": "fp64" if ff >= fh else "hbm", "kernel": "k_matvec_multi_partial<%d> + reduce (K4, %d right-hand "
            "sides)" % (min(nmv, 10), nmv), "achieved": tfs if ff >= fh else gbs,
            "peak": sustained if ff >= fh else hbm, "unit": "TFLOP/s" if ff >= fh else "GB/s", "frac": max(ff, fh),
            "hbm_gbs": gbs, "frac_hbm": fh, "fp64_tflops": tfs, "frac_fp64": ff, "ms": ms}


def nearfield_roofline(nf, nf_ms, peaks_fp64):
    """K3 against the FP64 pipe with the reference algorithm's work: every
    analytic call accurate_adaptive makes (assembly.cpp:548-605: the probe, then
    per visited node the node's own 7-point sum again plus its four children's —
    the device carries the parent's sub-cell value down, 28 calls per node)
    times F_analytic, plus the Gauss x Gauss 1/r pairs (YContext::gauss,
    assembly.cpp:504-543) times the Laplace pair probe."""
    pairs, _ = nf.info()
    dev_calls = nf.stats()[0]
    nodes = (dev_calls - 7 * pairs) / 28.0
    ref_calls = dev_calls + 7.0 * nodes
    gauss_pairs = pairs * 36  # 6-point rule on both triangles (cfg 3)
    work = ref_calls * F_ANALYTIC_FLOPS + gauss_pairs * F_PAIR_PROBE_FLOPS[False]
    achieved = work / (nf_ms * 1e-3) / 1e12
    burst, sustained, _, _ = peaks_fp64
    return {"bound": "fp64", "kernel": "k_nearfield_b (K3)", "achieved": achieved, "peak": sustained,
            "unit": "TFLOP/s", "frac": achieved / sustained, "frac_of_burst": achieved / burst,
            "reference_calls": ref_calls, "device_calls": dev_calls, "F_analytic_flops": F_ANALYTIC_FLOPS,
            "work": "reference analytic calls x F_analytic (canonical libdevice probe) + 36 Gauss 1/r pairs per "
                    "near pair x the Laplace probe; > 1 means the device formulation (solid angle, one log per "
                    "edge, carried parent values) needs fewer flops than the canonical one",
            "ncu_fp64_pipe_pct": profile_summary(3).get("k_nearfield_fp64_pipe_pct")}


def e2e_dense(g, torch, dev, cfg, pp, opts, n, nmv, xs, pairs_ref, steps, warmup, multi):
    """The same step through the public host API with HOST buffers: host side
    tables -> AssemblyPlan (gk_plan_create: host planning + table upload) ->
    gk_plan_assemble into the device-resident matrix [-> NearField] -> per
    vector: pinned x host->device, gk_matvec, y device->host (multi: all vectors
    host->device, one gk_matvec_multi, all results device->host).  Wall clock per
    step, everything inside; the matrix buffer is allocated once (the device
    memory the caller keeps A in)."""
    s = SPECS[cfg]
    space, dom, kern = pp["space"], pp["dom"], pp["kern"]
    A = torch.empty(n * n, dtype=torch.complex128, device=dev)
    xh = torch.tensor(np.asarray(xs, dtype=np.complex128).reshape(nmv, n)).pin_memory()
    yh = torch.empty((nmv, n), dtype=torch.complex128).pin_memory()
    xd = torch.empty((nmv, n), dtype=torch.complex128, device=dev)
    yd = torch.empty((nmv, n), dtype=torch.complex128, device=dev)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    h2d_tables = [0]

    def one(ev=None):
        t_a = time.perf_counter()
        plan = g.AssemblyPlan(dom, dom, space, kern, space, opts)
        h2d_tables[0] = plan.info()["device_bytes"]
        if ev:
            ev[2] = time.perf_counter() - t_a  # host planning + table upload
            ev[0].record(stream)
        plan.assemble(A.data_ptr(), n, sp)
        if cfg == 3:
            nf = g.NearField(dom, dom, space, "[1/r]", space)
            nf.compute(sp)
            nf.apply(A.data_ptr(), n, sp)
        if multi:
            xd.copy_(xh, non_blocking=True)
            g.matvec_multi(A.data_ptr(), n, n, n, xd.data_ptr(), n, yd.data_ptr(), n, nmv, sp)
            yh.copy_(yd, non_blocking=True)
        else:
            for i in range(nmv):
                xd[0].copy_(xh[i], non_blocking=True)
                g.matvec(A.data_ptr(), n, n, n, xd[0].data_ptr(), yd[0].data_ptr(), sp)
                yh[i].copy_(yd[0], non_blocking=True)
        if ev:
            ev[1].record(stream)
        torch.cuda.synchronize(dev)

    for _ in range(max(1, min(3, warmup))):
        one()
    ts = []
    evs = [[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True), 0.0] for _ in range(steps)]
    with ClockSampler(dev.index or 0) as clk:
        for i in range(steps):
            t = time.perf_counter()
            one(evs[i])
            ts.append(time.perf_counter() - t)
    del A
    torch.cuda.empty_cache()
    t = float(np.mean(ts))
    dev_ms = [e[0].elapsed_time(e[1]) for e in evs]
    return {"value": pairs_ref / t, "unit": "pairs/s", "h2d_bytes_per_step": int(h2d_tables[0] + 16 * n * nmv),
            "d2h_bytes_per_step": int(16 * n * nmv), "s_per_step": t, "s_per_step_median": float(np.median(ts)),
            "s_per_step_min": float(np.min(ts)), "s_per_step_max": float(np.max(ts)),
            "s_per_step_all": [round(x, 4) for x in ts],
            # where a step's time goes: the host planner + table upload, then the device work
            # (assembly, copies and matvecs, CUDA events), and the board's clocks over the leg
            "plan_s_all": [round(e[2], 4) for e in evs], "device_s_all": [round(x * 1e-3, 4) for x in dev_ms],
            "clocks": clk.summary(),
            "steps": steps,
            "path": "C-ABI through the host API: host mesh tables -> gk_plan_create (host plan + table upload) -> "
                    "gk_plan_assemble (device-resident A)%s -> %s; wall clock"
                    % (" -> gk_nearfield_create/compute/apply" if cfg == 3 else "",
                       "%d x pinned H2D, gk_matvec_multi, %d x D2H" % (nmv, nmv) if multi else
                       "%d x (x pinned H2D, gk_matvec, y D2H)" % nmv)}


def run_green(args, g, torch, dev, rank, world, dist, steps, warmup, peaks_fp64, with_cpu, with_e2e):
    """cfg 5: matrix-free Green matvec (K5).  A step is one fp64 matvec of the
    983,040 Gauss points against themselves; the fp32 variant is timed beside it."""
    s = SPECS[5]
    pp = product_problem(g, 5)
    pts, w, _ = g.quadrature(pp["dom"])
    pts = np.asarray(pts)
    q = np.asarray(w) * g.complex_normal(s["seed"], len(w))
    plan = g.GreenPlan(pts, pts, pp["kern"])
    info = plan.info()
    qd = torch.tensor(q, device=dev)
    y = torch.empty(len(w), dtype=torch.complex128, device=dev)
    stream = torch.cuda.current_stream(dev)
    res, clocks = {}, None
    for prec, label in ((g.FP64, "fp64"), (g.FP32, "fp32")):
        for _ in range(max(3, warmup)):
            plan.matvec(qd.data_ptr(), y.data_ptr(), prec, stream.cuda_stream)
        if dist:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(dev.index or 0) as clk:
            e0.record(stream)
            for _ in range(steps):
                plan.matvec(qd.data_ptr(), y.data_ptr(), prec, stream.cuda_stream)
            e1.record(stream)
            torch.cuda.synchronize(dev)
        if dist:
            dist.barrier()
        ms = max_over_ranks(e0.elapsed_time(e1) / steps, dist, dev)
        if label == "fp64":
            clocks = clk.summary()
        U = info["unique_targets"]
        res[label] = {"ms": ms, "pairs_per_s": world * len(w) ** 2 / (ms * 1e-3),
                      "unique_pairs_per_s": world * U * U / (ms * 1e-3)}
    if rank != 0:
        return None
    U = info["unique_targets"]
    helm = pp["k"] != 0.0
    evaluated = U * (U + 1) / 2 if info.get("symmetric") else U * U
    t = res["fp64"]["ms"] * 1e-3
    burst, sustained, sus_clk, _ = peaks_fp64
    achieved = evaluated * F_PAIR_PROBE_FLOPS[helm] / t / 1e12
    M = len(w)
    out = {
        "metric": METRIC_GREEN, "value": res["fp64"]["pairs_per_s"], "unit": "pairs/s", "n_gpus": world,
        "steps": steps, "warmup": warmup, "ms_per_step": res["fp64"]["ms"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64 (complex128); fp32 variant in detail",
        "data": "synthetic (seeded icosphere L7 Gauss nodes, SplitMix64/Box-Muller charges)",
        "config": config_dict(5, pp["nv"], pp["ne"], 0, M, pp["k"], pp["hbar"]) | {"unique": U,
                                                                                  "parallelism": f"replicas x{world}"},
        "detail": res, "info": info,
        "roofline": {"bound": "fp64", "kernel": "k_green64_sym (K5)", "achieved": achieved, "peak": sustained,
                     "unit": "TFLOP/s", "frac": achieved / sustained, "traffic": None,
                     "peak_source": "sustained DFMA+store FP64 peak measured in this run",
                     "peak_burst": burst, "frac_of_burst": achieved / burst,
                     "work": "evaluated unique pairs (%s) x %.0f flops/pair (probe F_pair)"
                             % ("symmetric: U(U+1)/2" if info.get("symmetric") else "U^2", F_PAIR_PROBE_FLOPS[helm])},
        "clocks": clocks,
        "gpu_launches": plan.launches(g.FP64) * steps,
    }
    if with_e2e:
        # host charges in, host potentials out, plan (host twin merge + upload) inside
        qh = torch.tensor(q).pin_memory()
        yh = torch.empty(M, dtype=torch.complex128).pin_memory()
        ts = []
        for it in range(max(2, min(steps, 5)) + 1):
            t0 = time.perf_counter()
            p2 = g.GreenPlan(pts, pts, pp["kern"])
            qd.copy_(qh, non_blocking=True)
            p2.matvec(qd.data_ptr(), y.data_ptr(), g.FP64, stream.cuda_stream)
            yh.copy_(y, non_blocking=True)
            torch.cuda.synchronize(dev)
            if it:
                ts.append(time.perf_counter() - t0)
            del p2
        tm = float(np.mean(ts))
        out["e2e"] = {"value": M * M / tm, "unit": "pairs/s", "h2d_bytes_per_step": int(16 * M + 24 * M),
                      "d2h_bytes_per_step": int(16 * M), "s_per_step": tm, "steps": len(ts),
                      "path": "GreenPlan(host points) + pinned charges H2D + gk_green_matvec + D2H; wall clock"}
    if with_cpu and world == 1:
        out["cpu_baseline"] = cpu_baseline(load_oracle(), 5, 8, threads=1)
    return out


# ---------------------------------------------------------------------------------
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch

    dist = None
    if args.impl == "b200" and torch.cuda.is_available():
        torch.cuda.set_device(local)  # before NCCL init, so each rank's communicator binds its own GPU
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl" if args.impl == "b200" else "gloo")
    if args.impl == "reference":
        return reference_arm(args, rank, world, dist)

    import paper_1804_00995_b200 as g

    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    peaks_fp64 = fp64_peaks(g, torch, dev, stream)
    if args.extras is None:
        extras = [2, 3, 5] if (args.config == 4 and world == 1) else []
    else:
        extras = [int(c) for c in args.extras.split(",") if c.strip() and c.strip() != "none"]
    others = {}
    for c in extras:
        if c == args.config:
            continue
        try:
            st = min(args.steps, 10)
            if c == 5:
                others[f"cfg{c}"] = run_green(args, g, torch, dev, rank, world, dist, st, 3, peaks_fp64,
                                              not args.no_cpu_baseline, not args.no_e2e)
            else:
                others[f"cfg{c}"] = run_dense(args, g, torch, dev, rank, world, dist, c, st, 3, peaks_fp64,
                                              not args.no_cpu_baseline, not args.no_e2e)
        except Exception as e:  # an extra line never takes the headline down
            others[f"cfg{c}"] = {"error": repr(e)}
        torch.cuda.synchronize(dev)
        torch.cuda.empty_cache()
    if args.config == 5:
        out = run_green(args, g, torch, dev, rank, world, dist, args.steps, args.warmup, peaks_fp64,
                        not args.no_cpu_baseline, not args.no_e2e)
    else:
        out = run_dense(args, g, torch, dev, rank, world, dist, args.config, args.steps, args.warmup, peaks_fp64,
                        not args.no_cpu_baseline, not args.no_e2e)
    if rank == 0:
        if others:
            out["other_configs"] = others
        print(json.dumps(out))
    if dist:
        dist.destroy_process_group()


def load_ref_module():
    """The reference's OWN sources (proj/src/{mesh,quadrature,kernels,femspace,
    assembly}.cpp) compiled against the Eigen-API shim into oracle/_ref/ by
    oracle/Makefile `ref` (test infrastructure; built in the build container,
    the .so travels to the GPU box).  None if it was not built."""
    import glob
    import importlib

    d = os.path.join(ROOT, "oracle", "_ref")
    if not glob.glob(os.path.join(d, "_ref*.so")):
        return None
    if d not in sys.path:
        sys.path.insert(0, d)
    return importlib.import_module("_ref")


def mem_available_bytes():
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except Exception:
        pass
    return 16 << 30


def reference_arm_compiled(args, R, cfg, threads=None, steps=None, warmup=None):
    """The reference's own bem_product (assembly.cpp:192-222, through bem_dense
    :313-320, single-threaded as written) on the box's host cores: each step,
    every worker thread runs the reference on its own contiguous slice of test
    triangles (the complete trial side), all threads at once; the step time is
    the wall time of that parallel sample extrapolated linearly in test
    quadrature points to the whole matrix, plus the step's stored matvecs on
    the rows the sample produced (numpy, all vectors in one product, scaled by
    rows).  Mesh, statistics and k come from the reference's own build_sphere /
    edge_stats (bit-identical to the product's, tests/test_ref_pins.py)."""
    from concurrent.futures import ThreadPoolExecutor

    s = SPECS[cfg]
    v, e = R.build_sphere(s["n"], 1.0)
    v, e = np.asarray(v), np.asarray(e)
    hbar = R.edge_stats(v, e)[2]
    k = 2 * math.pi / (10 * hbar) if s["helm"] else 0.0
    name = "[exp(ikr)/r]" if s["helm"] else "[1/r]"
    fam = 1 if s["fam"] == "P1" else 0
    ne, nv, g = len(e), len(v), s["gauss"]
    N = nv if fam == 1 else ne
    M = ne * g
    R.rule(g)  # the reference's rule cache (a std::map) is filled before the threads start
    threads = threads or os.cpu_count() or 1
    steps = args.steps if steps is None else steps
    warmup = args.warmup if warmup is None else warmup
    # per-thread slice: about 96 test triangles (288 points, well under the
    # reference's 1024-point chunk) — a few seconds of single-core work
    per = max(1, min(96, ne // threads))
    per_thread_bytes = 16.0 * (per * g * M + per * g * N + per * 3 * N) * 1.3
    threads = max(1, min(threads, int(0.5 * mem_available_bytes() / per_thread_bytes)))
    nslices = max(1, ne // per)
    xs = np.stack([complex_normal_ref(s["seed"], N * s["nmv"])[i * N:(i + 1) * N] for i in range(s["nmv"])]
                  if not s["real_x"] else [np.asarray(ref_normal(s["seed"], N), dtype=np.complex128)])

    def slice_mesh(j):
        t0 = (j * 7919) % nslices * per  # slices spread over the mesh, cycled
        sub = e[t0:t0 + per]
        if fam == 0:
            return v, sub, None
        used, inv = np.unique(sub.ravel(), return_inverse=True)  # P1: the slice's own vertices
        return v[used], inv.reshape(sub.shape).astype(np.int32), used

    def work(j):
        vx, ex, used = slice_mesh(j)
        t = time.perf_counter()
        A = R.bem_dense(vx, ex, g, fam, v, e, g, fam, name, k, 1e15)
        return A, time.perf_counter() - t

    pool = ThreadPoolExecutor(max_workers=threads)
    step_id = [0]

    def one_step():
        ids = [step_id[0] * threads + i for i in range(threads)]
        step_id[0] += 1
        t0 = time.perf_counter()
        res = list(pool.map(work, ids))
        wall = time.perf_counter() - t0
        rows = np.concatenate([r[0] for r in res], axis=0)  # sample rows x N
        t1 = time.perf_counter()
        Y = rows @ xs.T  # the step's matvecs on the sampled rows
        t_mv = time.perf_counter() - t1
        assert np.isfinite(Y).all()
        pts = threads * per * g
        return wall * M / pts + t_mv * N / rows.shape[0], wall, t_mv, rows.shape[0]

    one_step()  # warm-up (page faults, thread start)
    for _ in range(max(0, min(warmup, 1) - 1)):
        one_step()
    ests, walls = [], []
    for _ in range(steps):
        est, wall, t_mv, nrows = one_step()
        ests.append(est)
        walls.append(wall)
    pool.shutdown()
    est = float(np.mean(ests))
    sample = (f"the reference's own bem_dense/bem_product (proj/src, compiled unchanged against the Eigen-API shim, "
              f"oracle/_ref) on {threads} host threads at once, each on a slice of {per} test triangles "
              f"({per * g} x points) x all {M} trial points ({float(np.mean(walls)):.1f} s wall per step), "
              f"+ {s['nmv']} matvecs on the sampled rows (numpy); extrapolated linearly in x points / rows "
              f"to the full {N} x {N} step")
    return dict(value=M * M / est, est=est, sample=sample, threads=threads, N=N, M=M, k=k, hbar=hbar, nv=nv, ne=ne)


def complex_normal_ref(seed, n):
    """complex_normal without the product: the oracle's SplitMix64 stream."""
    return complex_normal_np(load_oracle(), seed, n)


def ref_normal(seed, n):
    o = load_oracle()
    u = np.asarray(o.uniform01_stream(seed, 2 * ((n + 1) // 2)))
    r = np.sqrt(-2.0 * np.log(1.0 - u[0::2]))
    t = 2.0 * np.pi * u[1::2]
    z = np.empty(2 * len(r))
    z[0::2] = r * np.cos(t)
    z[1::2] = r * np.sin(t)
    return z[:n]


def reference_arm(args, rank, world, dist):
    """The reference's CPU path on the host cores: the oracle (C++ restatement
    of bem_product / regularize / zgemv / the matrix-free loop; the reference
    cannot be built here) with all host threads.  Nothing from the product is
    imported.  Each step is one 1024-point x chunk (cycling over 8 uniformly
    spaced chunks) + the step's matvecs on its rows, extrapolated to the full
    step; cfg 5: one block of 96 targets."""
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    cfg = args.config
    s = SPECS[cfg]
    R = load_ref_module() if cfg in (1, 2, 4) else None  # cfg 3's 6-point rule and cfg 5's matrix-free
    # loop are not in the reference: those configs time the oracle restatement (kind "port")
    if R is not None:
        r = reference_arm_compiled(args, R, cfg)
        cfgd = config_dict(cfg, r["nv"], r["ne"], r["N"], r["M"], r["k"], r["hbar"]) | {
            "parallelism": f"replicas x{world}"}
        value = r["value"]
        out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["est"] * 1e3, "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "f64 (complex128)",
               "data": "synthetic (seeded icosphere mesh per BASELINE config, SplitMix64/Box-Muller vectors)",
               "config": cfgd,
               "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": r["threads"], "kind": "reference",
                                "sample": r["sample"]},
               "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        assert "paper_1804_00995_b200" not in sys.modules, "the reference arm must not load the product"
        print(json.dumps(out))
        if dist:
            dist.destroy_process_group()
        return
    o = load_oracle()
    P = oracle_problem(o, cfg)
    threads = os.cpu_count() or 1
    if cfg == 5:
        pts, w, _ = o.quadrature(P["v"], P["e"], P["g"])
        pts, w = np.asarray(pts), np.asarray(w)
        q = w * complex_normal_np(o, s["seed"], len(w))
        lo, hi = pts.min(axis=0), pts.max(axis=0)
        eps = 1e-12 * float(np.linalg.norm(hi - lo))
        blocks = np.linspace(0, P["M"] - 96, 8).astype(np.int64)
        cpu_green_step(o, P, threads, np.arange(4), eps, q)  # warm-up
        ests = []
        for i in range(args.steps):
            ids = np.arange(blocks[i % 8], blocks[i % 8] + 96)
            ests.append(cpu_green_step(o, P, threads, ids, eps, q)[0])
        est = float(np.mean(ests))
        sample = f"oracle matrix-free Green matvec, 96 targets x {P['M']} sources per step (8 uniformly spaced blocks)"
        metric = METRIC_GREEN
        N = 0
    else:
        xs = [complex_normal_np(o, s["seed"], P["N"] * s["nmv"])[i * P["N"]:(i + 1) * P["N"]] for i in range(s["nmv"])]
        chunks, npts = chunk_rows(o, P, 8)
        o.bem_dense(P["v"], P["e"], P["g"], P["fam"], P["v"], P["e"], P["g"], P["fam"], P["name"], P["k"],
                    rows=chunks[0][:4], threads=threads, cap=1e15)  # warm-up
        ests = []
        for i in range(args.steps):
            ests.append(cpu_dense_step(o, P, cfg, chunks[i % 8], npts[i % 8], threads, xs)[0])
        est = float(np.mean(ests))
        sample = (f"oracle bem_product restatement{' + regularize' if cfg == 3 else ''} + {s['nmv']} zgemv on the "
                  f"complete rows of one 1024-point x chunk per step (8 uniformly spaced chunks, cycled), "
                  f"extrapolated to the full step")
        metric = METRIC
        N = P["N"]
    value = P["M"] ** 2 / est
    cfgd = config_dict(cfg, P["nv"], P["ne"], N, P["M"], P["k"], P["hbar"]) | {"parallelism": f"replicas x{world}"}
    out = {"impl": "reference", "metric": metric, "value": value, "unit": "pairs/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": est * 1e3, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64 (complex128)",
           "data": "synthetic (seeded icosphere mesh per BASELINE config, SplitMix64/Box-Muller vectors)",
           "config": cfgd,
           "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": threads, "kind": "port", "sample": sample},
           "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
