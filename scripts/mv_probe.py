"""Stored matvec probe: y = A x on an n x n complex128 device matrix
(uninitialised contents do not change the traffic), for ncu dram__bytes
captures of k_matvec_partial / k_matvec_multi.

  python scripts/mv_probe.py --n 81920 [--nrhs 10]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_00995_b200 as g  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=81920)
p.add_argument("--nrhs", type=int, default=1)
p.add_argument("--reps", type=int, default=1)
a = p.parse_args()
n = a.n
A = torch.zeros(n * n, dtype=torch.complex128, device="cuda")
X = torch.ones(a.nrhs * n, dtype=torch.complex128, device="cuda")
Y = torch.empty(a.nrhs * n, dtype=torch.complex128, device="cuda")
s = torch.cuda.current_stream().cuda_stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(a.reps + 1):
    if rep == 1:
        e0.record()
    if a.nrhs == 1:
        g.matvec(A.data_ptr(), n, n, n, X.data_ptr(), Y.data_ptr(), s)
    else:
        g.matvec_multi(A.data_ptr(), n, n, n, X.data_ptr(), n, Y.data_ptr(), n, a.nrhs, s)
e1.record()
torch.cuda.synchronize()
if a.reps:
    ms = e0.elapsed_time(e1) / a.reps
    print(f"n={n} nrhs={a.nrhs}: {ms:.3f} ms, {16.0 * n * n / ms / 1e6:.1f} GB/s of A")
