"""Breakdown of the cfg-4 e2e step (bench.py e2e_dense) with GK_TIMING=1:
AssemblyPlan (host plan + upload), assemble, matvec_multi with host vectors."""
import math
import os
import sys
import time

import numpy as np
import torch

os.environ.setdefault("GK_TIMING", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_00995_b200 as g  # noqa: E402

m = g.build_sphere(40962, 1.0)
dom = g.make_domain(m, 3)
sp = g.make_fem(m, "P0")
k = 2 * math.pi / (10 * g.edge_stats(m).mean_len)
kern = g.green_kernel("[exp(ikr)/r]", k)
o = g.BemOptions()
o.memory_cap_bytes = 10 ** 15
n = sp.free_count()
A = torch.empty(n * n, dtype=torch.complex128, device="cuda")
xh = torch.tensor(np.asarray(g.complex_normal(3, 10 * n)).reshape(10, n)).pin_memory()
yh = torch.empty((10, n), dtype=torch.complex128).pin_memory()
xd = torch.empty((10, n), dtype=torch.complex128, device="cuda")
yd = torch.empty((10, n), dtype=torch.complex128, device="cuda")
s = torch.cuda.current_stream().cuda_stream
print("nproc", os.cpu_count(), flush=True)
for it in range(int(os.environ.get("E2E_STEPS", "4"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = g.AssemblyPlan(dom, dom, sp, kern, sp, o)
    t1 = time.perf_counter()
    plan.assemble(A.data_ptr(), n, s)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    xd.copy_(xh, non_blocking=True)
    g.matvec_multi(A.data_ptr(), n, n, n, xd.data_ptr(), n, yd.data_ptr(), n, 10, s)
    yh.copy_(yd, non_blocking=True)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    del plan
    t4 = time.perf_counter()
    print(f"step {it}: plan {1e3 * (t1 - t0):.1f} assemble {1e3 * (t2 - t1):.1f} matvecs {1e3 * (t3 - t2):.1f} "
          f"destroy {1e3 * (t4 - t3):.1f} total {1e3 * (t4 - t0):.1f} ms", flush=True)
