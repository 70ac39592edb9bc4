#!/usr/bin/env python
"""bench.py — driver-contract benchmark for the B200 dense BEM hot path.

Default workload (BASELINE.json configs[1], "cfg2"): unit-sphere icosphere L5
(10242 vertices, 20480 triangles), P1 Lagrange, 3-point (edge-midpoint) rule,
Helmholtz single layer with k = 2 pi / (10 hbar); one step = dense assembly of
the 10242 x 10242 complex128 matrix (K1+K2, device-resident tables) followed
by one stored matvec y = A x (K4, x complex N(0,1) from seed 1).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--config 1|2|3|4|5]

Metric: reference-equivalent quadrature-pair kernel evaluations per second
(M_x * M_y per assembly / step time), plus matrix entries/s and matvec GB/s.
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
# counters (profiles/r01_fpair_probe.txt):
#  - canonical probe: the reference formula kernels.cpp:94-114 with
#    libdevice sqrt/sin/cos/division + one complex x real accumulate:
#    43 DFMA + 13 DMUL + 7 DADD = 106 flops/pair (DFMA = 2 flops);
#  - production formula: SASS count of k_assemble's pair loop (cuobjdump, P1
#    cfg 2, y-side accumulation included): 23 DFMA + 7 DMUL + 4 DADD = 57
#    flops/pair (59 before the degree-6 cos polynomial); Laplace: 5 DFMA + 4 DMUL + 5 DADD = 19.
# Laplace ("[1/r]", cfg 1) probe: 11 FP64 instructions + accumulate = 23 flops.
F_PAIR_PROBE_FLOPS = {True: 106.0, False: 23.0}
F_PAIR_PROD_FLOPS = {True: 57.0, False: 19.0}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["b200", "reference"], default="b200")
    p.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    return p.parse_args()


# ---------------------------------------------------------------------------------
def config_problem(g, cfg):
    """Mesh/space/kernel of a BASELINE config."""
    spec = {
        1: dict(n=642, gauss=3, fam="P1", helm=False, perturb=None, seed=0, real_x=True),
        2: dict(n=10242, gauss=3, fam="P1", helm=True, perturb=None, seed=1, real_x=False),
        3: dict(n=10242, gauss=6, fam="P0", helm=True, perturb=2, seed=1, real_x=False),
        4: dict(n=40962, gauss=3, fam="P0", helm=True, perturb=None, seed=3, real_x=False),
        5: dict(n=163842, gauss=3, fam="points", helm=True, perturb=None, seed=4, real_x=False),
    }[cfg]
    mesh = g.build_sphere(spec["n"], 1.0)
    if spec["perturb"] is not None:
        mesh = g.perturb_radial(mesh, spec["perturb"], 0.02)
    hbar = g.edge_stats(mesh).mean_len
    k = 2 * math.pi / (10 * hbar) if spec["helm"] else 0.0
    name = "[exp(ikr)/r]" if spec["helm"] else "[1/r]"
    dom = g.make_domain(mesh, spec["gauss"])
    space = g.make_fem(mesh, spec["fam"]) if spec["fam"] != "points" else None
    return spec, mesh, dom, space, g.green_kernel(name, k), k, hbar, name


def workload_name(cfg, spec, mesh):
    nv, ne = mesh.vertex_count(), mesh.element_count()
    return {
        1: f"cfg1: Laplace single layer, P1, 3-pt, icosphere L3 ({nv} v/{ne} t), 642^2 real-valued complex128 + matvec",
        2: f"cfg2: Helmholtz single layer, P1, 3-pt, icosphere L5 ({nv} v/{ne} t), 10242^2 complex128 + matvec",
        3: f"cfg3: Helmholtz single layer, P0, 6-pt, perturbed L5 ({ne} t), 20480^2 complex128 + matvec (dense part)",
        4: f"cfg4: Helmholtz single layer, P0, 3-pt, icosphere L6 ({ne} t), 81920^2 complex128 (107 GB) + 10 matvecs",
        5: f"cfg5: matrix-free Helmholtz Green matvec, 983040 points of L7 ({ne} t)",
    }[cfg]


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
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            return json.load(f).get(f"cfg{cfg}", {})
    except Exception:
        return {}


def profile_traffic(cfg):
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    return profile_summary(cfg).get("k_assemble_dram_bytes_per_launch")


# ---------------------------------------------------------------------------------
def cpu_sample_rows(oracle, mesh, gauss, fam, target_points):
    """Evenly spaced test dofs whose supporting x points total ~target_points."""
    start, dof, _ = oracle.eval_rows(mesh.vertices, mesh.elements, fam, gauss)
    start = np.asarray(start)
    dof = np.asarray(dof)
    ndof = mesh.vertex_count() if fam == 1 else mesh.element_count()
    per_dof = np.bincount(dof, minlength=ndof)
    count = max(1, int(target_points / max(1.0, per_dof.mean())))
    rows = sorted(set(np.linspace(0, ndof - 1, count).astype(int).tolist()))
    sel = np.isin(dof, rows)
    pt_of = np.repeat(np.arange(len(start) - 1), np.diff(start))
    npts = len(np.unique(pt_of[sel]))
    return rows, npts


def run_cpu(oracle, mesh, spec, k, name, rows, threads, cap=1e13):
    fam = 1 if spec["fam"] == "P1" else 0
    t = time.perf_counter()
    oracle.bem_dense(mesh.vertices, mesh.elements, spec["gauss"], fam, mesh.vertices, mesh.elements, spec["gauss"],
                     fam, name, k, rows=rows, threads=threads, cap=cap)
    return time.perf_counter() - t


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

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    spec, mesh, dom, space, kern, k, hbar, kname = config_problem(g, args.config)
    if args.config == 5:
        return bench_green(args, g, torch, dev, rank, world, dist, spec, mesh, dom, kern, k, hbar)

    opts = g.BemOptions()
    opts.memory_cap_bytes = 10 ** 15  # the reference's 8e9 cap refuses cfg 3/4 (SURVEY trap 5)
    plan = g.AssemblyPlan(dom, dom, space, kern, space, opts)
    info = plan.info()
    n = info["rows"]
    A = torch.empty(n * n, dtype=torch.complex128, device=dev)
    nmv = 10 if args.config == 4 else 1
    # cfg 4: ten vectors drawn consecutively from the seed-3 stream
    xs = g.normal(spec["seed"], n) if spec["real_x"] else g.complex_normal(spec["seed"], nmv * n)
    X = torch.tensor(np.asarray(xs, dtype=np.complex128).reshape(nmv, n), device=dev)
    y = torch.empty(n, dtype=torch.complex128, device=dev)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    # cfg 3: "including the near-field singular correction" -> K3 inside the step
    nf = g.NearField(dom, dom, space, "[1/r]", space) if args.config == 3 else None
    launches_per_step = plan.launches() + nmv * g.matvec_launches(n, n) + (3 if nf else 0)

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        plan.assemble(A.data_ptr(), n, sp)
        if nf:
            if ev:
                ev[3].record(stream)
            nf.compute(sp)
            nf.apply(A.data_ptr(), n, sp)
        if ev:
            ev[1].record(stream)
        for i in range(nmv):
            g.matvec(A.data_ptr(), n, n, n, X[i].data_ptr(), y.data_ptr(), sp)
        if ev:
            ev[2].record(stream)

    fp64_peak_gflops = g.diag_fp64_peak(20000, sp)  # DFMA microbenchmark, this run
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize(dev)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        t0.record(stream)
        for i in range(args.steps):
            step(evs[i])
        t1.record(stream)
        torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    total_ms = t0.elapsed_time(t1)
    if nf:
        nf_ms = float(np.mean([e[3].elapsed_time(e[1]) for e in evs]))
        asm_ms = float(np.mean([e[0].elapsed_time(e[3]) for e in evs]))
    else:
        nf_ms = None
        asm_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in evs]))
    mv_ms = float(np.mean([e[1].elapsed_time(e[2]) for e in evs])) / nmv
    nf_2h = None
    if nf:
        # BASELINE words cfg 3's near field as "pairs closer than 2 hbar"; the
        # reference's rule (used in the step) is 3 max circumradius (SURVEY trap 3).
        # The 2-hbar mode is timed beside it, outside the step.
        nf2 = g.NearField(dom, dom, space, "[1/r]", space, g.NEAR_2HBAR, hbar)
        nf2.compute(sp)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        nf2.compute(sp)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        nf_2h = {"ms": e0.elapsed_time(e1), "pairs": nf2.info()[0], "analytic_calls": nf2.stats()[0]}
    total_ms = max_over_ranks(total_ms, dist, dev)
    ms_step = total_ms / args.steps
    pairs_ref = info["pairs_reference"]
    value = aggregate_value(pairs_ref, world, ms_step)

    out = None
    if rank == 0:
        peaks = measured_peaks()
        hbm = peaks.get("hbm_gbs", HBM_FALLBACK_GBS)
        helm = k != 0.0
        alg_flops = info["pairs_unique"] * F_PAIR_PROBE_FLOPS[helm]
        achieved = alg_flops / (asm_ms * 1e-3) / 1e12
        achieved_prod = info["pairs_unique"] * F_PAIR_PROD_FLOPS[helm] / (asm_ms * 1e-3) / 1e12
        exec_prod = info["pairs_evaluated"] * F_PAIR_PROD_FLOPS[helm] / (asm_ms * 1e-3) / 1e12
        peak = fp64_peak_gflops / 1e3
        mv_bytes = 16.0 * n * n + 32.0 * n
        clocks = clk.summary()
        out = {
            "metric": "quadrature-pair kernel evals/s (reference-equivalent M_x*M_y per assembly, fp64)",
            "value": value,
            "unit": "pairs/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_step,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64 (complex128)",
            "data": "synthetic (seeded icosphere mesh, SplitMix64/Box-Muller vectors)",
            "config": {"workload": workload_name(args.config, spec, mesh), "N": n, "M": int(math.isqrt(pairs_ref)),
                       "k": k, "hbar": hbar, "parallelism": f"replicas x{world}",
                       "l2": "inputs larger than L2: A = %.2f GB written+read per step; plan tables %.1f MB"
                             % (16 * n * n / 1e9, info["device_bytes"] / 1e6)},
            "entries_per_s": world * n * n / (ms_step * 1e-3),
            "assembly_ms": asm_ms,
            "nearfield_ms": nf_ms,
            "nearfield": (dict(zip(("pairs", "entries"), nf.info())) | {"analytic_calls": nf.stats()[0], "rule": "ref"})
                         if nf else None,
            "nearfield_2hbar": nf_2h,
            "matvec_ms": mv_ms,
            "matvec_gbs": mv_bytes / (mv_ms * 1e-3) / 1e9,
            "unique_pairs_per_s": info["pairs_unique"] / (asm_ms * 1e-3),
            "pairs_evaluated_per_unique": info["pairs_evaluated"] / info["pairs_unique"],
            "roofline": {"bound": "fp64", "kernel": "k_assemble (K1+K2)", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak, "traffic": profile_traffic(args.config),
                         "peak_source": "DFMA microbenchmark measured in this run (MEASURED_PEAKS.json has no FP64)",
                         "work": "pairs_unique (twins merged, symmetric half) x %.0f flops/pair = canonical "
                                 "libdevice probe F_pair (SURVEY 8d)" % F_PAIR_PROBE_FLOPS[helm],
                         "frac_production_formula": achieved_prod / peak,
                         "frac_executed_pairs_production_formula": exec_prod / peak,
                         "ncu_fp64_pipe_pct": profile_summary(args.config).get("fp64_pipe_pct"),
                         "ncu_sfu_xu_pipe_pct": profile_summary(args.config).get("xu_pipe_pct")},
            "roofline_matvec": {"bound": "hbm", "achieved": mv_bytes / (mv_ms * 1e-3) / 1e9, "peak": hbm,
                                "unit": "GB/s", "frac": mv_bytes / (mv_ms * 1e-3) / 1e9 / hbm,
                                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback"},
            "clocks": clocks,
            "gpu_launches": launches_per_step * args.steps,
        }
        if not args.no_e2e and args.config in (1, 2):
            out["e2e"] = e2e_dense(g, torch, dom, space, kern, opts, n, pairs_ref, steps=max(2, min(args.steps, 3)))
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(spec, mesh, k, kname, ms_step)
    if rank == 0:
        print(json.dumps(out))
    if dist:
        dist.destroy_process_group()


def e2e_dense(g, torch, dom, space, kern, opts, n, pairs_ref, steps):
    """Same metric through the public drop-in (gk_bem_dense): host mesh tables in,
    host (pinned) matrix out, every copy inside the timed region."""
    host = torch.empty(n * n, dtype=torch.complex128, pin_memory=True)
    g.bem_dense_into(dom, dom, space, kern, space, opts, host.data_ptr(), n)  # warm-up
    ts = []
    h2d = 0
    for _ in range(steps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        h2d = g.bem_dense_into(dom, dom, space, kern, space, opts, host.data_ptr(), n)
        ts.append(time.perf_counter() - t)
    t = float(np.median(ts))
    return {"value": pairs_ref / t, "unit": "pairs/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": 16 * n * n, "s_per_step": t,
            "path": "gk_bem_dense (C-ABI, host sides -> pinned host matrix; column slabs streamed: tables built ahead, D2H overlapped)"}


def cpu_baseline(spec, mesh, k, name, gpu_ms_step):
    from tests._support import load_oracle

    oracle = load_oracle()
    fam = 1 if spec["fam"] == "P1" else 0
    M = mesh.element_count() * spec["gauss"]
    rows, npts = cpu_sample_rows(oracle, mesh, spec["gauss"], fam, target_points=min(M, 1536))
    secs = run_cpu(oracle, mesh, spec, k, name, rows, threads=1)
    extra = ""
    if spec["fam"] == "P0" and spec["perturb"] is not None:  # cfg 3: the step includes regularize
        t0 = time.perf_counter()
        oracle.regularize(mesh.vertices, mesh.elements, spec["gauss"], 0, mesh.vertices, mesh.elements,
                          spec["gauss"], 0, "[1/r]", 0, 0.0, list(rows), 1)
        secs += time.perf_counter() - t0
        extra = " + regularize of those test elements"
    pairs = npts * M
    return {"value": pairs / secs, "unit": "pairs/s", "cores": 1, "kind": "port",
            "sample": f"oracle bem_product restatement, {len(rows)} complete test rows ({npts} x-points x {M} "
                      f"y-points = {pairs:.3g} pairs){extra} in {secs:.1f} s, 1 thread (reference concurrency)"}


def reference_arm(args, rank, world, dist):
    """The reference's CPU path timed on the host cores: the oracle (C++
    restatement, the reference cannot be built here) with all host threads."""
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    import paper_1804_00995_b200 as g
    from tests._support import load_oracle

    oracle = load_oracle()
    spec, mesh, dom, space, kern, k, hbar, kname = config_problem(g, args.config)
    threads = os.cpu_count() or 1
    if args.config == 5:
        return reference_arm_green(args, g, oracle, spec, mesh, dom, k, kname, threads, world, dist)
    fam = 1 if spec["fam"] == "P1" else 0
    M = mesh.element_count() * spec["gauss"]
    rows, npts = cpu_sample_rows(oracle, mesh, spec["gauss"], fam, target_points=min(M, 2048))
    for _ in range(max(1, args.warmup)):
        run_cpu(oracle, mesh, spec, k, kname, rows[:8], threads)
    ts = [run_cpu(oracle, mesh, spec, k, kname, rows, threads) for _ in range(args.steps)]
    t = float(np.mean(ts))
    if args.config == 3:
        # cfg 3's step includes the near-field correction: the reference's
        # regularize (assembly.cpp:609-697) for the same test elements (P0: row = element)
        nt = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            oracle.regularize(mesh.vertices, mesh.elements, spec["gauss"], 0, mesh.vertices, mesh.elements,
                              spec["gauss"], 0, "[1/r]", 0, 0.0, list(rows), threads)
            nt.append(time.perf_counter() - t0)
        t += float(np.mean(nt))
    value = npts * M / t
    out = {"impl": "reference", "metric": "quadrature-pair kernel evals/s (reference-equivalent M_x*M_y per assembly, fp64)",
           "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "f64 (complex128)", "data": "synthetic",
           "config": {"workload": workload_name(args.config, spec, mesh), "N": space.free_count() if space else None},
           "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": threads, "kind": "port",
                            "sample": f"oracle bem_product restatement (OpenMP over trial columns), {len(rows)} "
                                      f"complete test rows = {npts} x-points x {M} y-points per step"
                                      + (" + regularize of those test elements" if args.config == 3 else "")},
           "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    if dist:
        dist.destroy_process_group()


def reference_arm_green(args, g, oracle, spec, mesh, dom, k, kname, threads, world, dist):
    """cfg 5 reference arm: the oracle's matrix-free Green matvec (the reference's
    evaluate_blocks(mask=true) x weighted charges) on a sample of targets."""
    pts, w, _ = g.quadrature(dom)
    q = np.asarray(w) * g.complex_normal(spec["seed"], len(w))
    M = len(w)
    ids = list(range(0, M, M // 96))[:96]
    lo, hi = np.asarray(pts).min(axis=0), np.asarray(pts).max(axis=0)
    eps = 1e-12 * float(np.linalg.norm(hi - lo))  # singular_guard_radius (kernels.cpp:14-19)
    oracle.green_matvec(kname, k, pts, pts, q, eps, ids[:4], threads)  # warm-up
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.green_matvec(kname, k, pts, pts, q, eps, ids, threads)
        ts.append(time.perf_counter() - t0)
    t = float(np.mean(ts))
    value = len(ids) * M / t
    out = {"impl": "reference", "metric": "matrix-free Green matvec pair evals/s (reference-equivalent M^2 per matvec, fp64)",
           "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "f64 (complex128)", "data": "synthetic",
           "config": {"workload": "cfg5: matrix-free Helmholtz Green matvec, 983040 targets = sources", "M": M},
           "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": threads, "kind": "port",
                            "sample": f"oracle Green matvec, {len(ids)} targets x {M} sources per step"},
           "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    if dist:
        dist.destroy_process_group()


def bench_green(args, g, torch, dev, rank, world, dist, spec, mesh, dom, kern, k, hbar):
    """cfg 5: matrix-free Green matvec (K5).  A step is one fp64 matvec of the
    983,040 Gauss points against themselves; the fp32 variant is timed beside it."""
    pts, w, _ = g.quadrature(dom)
    q = np.asarray(w) * g.complex_normal(spec["seed"], len(w))
    plan = g.GreenPlan(pts, pts, kern)
    info = plan.info()
    qd = torch.tensor(q, device=dev)
    y = torch.empty(len(w), dtype=torch.complex128, device=dev)
    stream = torch.cuda.current_stream(dev)
    fp64_peak_gflops = g.diag_fp64_peak(20000, stream.cuda_stream)
    res = {}
    clocks = None
    for prec, label in ((g.FP64, "fp64"), (g.FP32, "fp32")):
        for _ in range(max(3, args.warmup)):
            plan.matvec(qd.data_ptr(), y.data_ptr(), prec, stream.cuda_stream)
        if dist:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(int(os.environ.get("LOCAL_RANK", 0))) as clk:
            e0.record(stream)
            for _ in range(args.steps):
                plan.matvec(qd.data_ptr(), y.data_ptr(), prec, stream.cuda_stream)
            e1.record(stream)
            torch.cuda.synchronize(dev)
        if dist:
            dist.barrier()
        ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, dist, dev)
        if label == "fp64":
            clocks = clk.summary()
        U = info["unique_targets"]
        res[label] = {"ms": ms, "pairs_per_s": world * len(w) ** 2 / (ms * 1e-3),
                      "unique_pairs_per_s": world * U * U / (ms * 1e-3)}
    if rank == 0:
        U = info["unique_targets"]
        helm = k != 0.0
        # evaluated pairs: the symmetric path evaluates each unordered unique pair once
        evaluated = U * (U + 1) / 2 if info.get("symmetric") else U * U
        t = res["fp64"]["ms"] * 1e-3
        peak = fp64_peak_gflops / 1e3
        achieved = evaluated * F_PAIR_PROBE_FLOPS[helm] / t / 1e12
        out = {
            "metric": "matrix-free Green matvec pair evals/s (reference-equivalent M^2 per matvec, fp64)",
            "value": res["fp64"]["pairs_per_s"], "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["fp64"]["ms"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64 (complex128); fp32 variant in detail",
            "data": "synthetic (seeded icosphere L7 Gauss nodes, SplitMix64/Box-Muller charges)",
            "config": {"workload": "cfg5: matrix-free Helmholtz Green matvec, 983040 targets = sources (icosphere L7, "
                                   "3-pt), self-interaction masked", "M": len(w), "unique": U, "k": k, "hbar": hbar,
                       "parallelism": f"replicas x{world}",
                       "l2": "sources re-streamed from L2 per tile; no matrix (matrix-free)"},
            "detail": res, "info": info,
            "roofline": {"bound": "fp64", "kernel": "k_green64_sym (K5)", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak, "traffic": None,
                         "peak_source": "DFMA microbenchmark measured in this run",
                         "work": "evaluated unique pairs (%s) x %.0f flops/pair (probe F_pair)"
                                 % ("symmetric: U(U+1)/2" if info.get("symmetric") else "U^2",
                                    F_PAIR_PROBE_FLOPS[helm])},
            "clocks": clocks,
            "gpu_launches": plan.launches(g.FP64) * args.steps,
        }
        print(json.dumps(out))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
