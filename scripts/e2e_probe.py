"""Breakdown of the one-shot gk_bem_dense call (cfg 2) with GK_TIMING=1."""
import os
import time

import numpy as np
import torch

os.environ.setdefault("GK_TIMING", "1")
import paper_1804_00995_b200 as g  # noqa: E402

m = g.build_sphere(10242, 1.0)
dom = g.make_domain(m, 3)
sp = g.make_fem(m, "P1")
k = 2 * np.pi / (10 * g.edge_stats(m).mean_len)
kern = g.green_kernel("[exp(ikr)/r]", k)
n = sp.free_count()
host = torch.empty(n * n, dtype=torch.complex128, pin_memory=True)
print("nproc", os.cpu_count(), "loadavg", os.getloadavg(), flush=True)
for it in range(int(os.environ.get("CALLS", "3"))):
    torch.cuda.synchronize()
    t = time.perf_counter()
    g.bem_dense_into(dom, dom, sp, kern, sp, g.BemOptions(), host.data_ptr(), n)
    print(f"call {it}: {1e3 * (time.perf_counter() - t):.2f} ms", flush=True)
for it in range(int(os.environ.get("PAGEABLE_CALLS", "2"))):
    t = time.perf_counter()
    A = g.bem_dense(dom, dom, sp, kern, sp)
    print(f"pageable call {it} (bem_dense -> new numpy matrix): {1e3 * (time.perf_counter() - t):.2f} ms", flush=True)
    del A
dev = torch.empty(n * n, dtype=torch.complex128, device="cuda")
for it in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    host.copy_(dev, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"plain D2H 1.68 GB: {1e3 * dt:.2f} ms = {16 * n * n / dt / 1e9:.1f} GB/s", flush=True)
