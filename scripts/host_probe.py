"""Host-side facts on the GPU box: cores, memcpy bandwidth (1 and N threads), pinned D2H of half a matrix."""
import os
import threading
import time

import numpy as np
import torch

print("nproc", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)), flush=True)
n = 10242
a = np.empty(n * n * 2, dtype=np.float64)
b = np.empty_like(a)
a[:] = 1.0
b[:] = 0.0
for nt in (1, 4, 8, 16):
    chunks = np.array_split(np.arange(a.size), nt)
    def work(c):
        b[c[0]:c[-1] + 1] = a[c[0]:c[-1] + 1]
    best = 1e9
    for _ in range(3):
        th = [threading.Thread(target=work, args=(c,)) for c in chunks]
        t = time.perf_counter()
        [x.start() for x in th]
        [x.join() for x in th]
        best = min(best, time.perf_counter() - t)
    print(f"host memcpy {a.nbytes/1e9:.2f} GB, {nt} threads: {a.nbytes/best/1e9:.1f} GB/s", flush=True)
dev = torch.empty(n * n, dtype=torch.complex128, device="cuda")
host = torch.empty(n * n, dtype=torch.complex128, pin_memory=True)
for frac in (1.0, 0.5):
    m = int(n * n * frac)
    for _ in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        host[:m].copy_(dev[:m], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"pinned D2H {16*m/1e9:.2f} GB: {1e3*dt:.2f} ms = {16*m/dt/1e9:.1f} GB/s", flush=True)
pageable = np.empty(n * n * 2, dtype=np.float64)
pageable[:] = 0
t = time.perf_counter()
torch.from_numpy(pageable).view(torch.complex128).copy_(dev)
torch.cuda.synchronize()
dt = time.perf_counter() - t
print(f"pageable D2H 1.68 GB: {1e3*dt:.2f} ms = {16*n*n/dt/1e9:.1f} GB/s", flush=True)
