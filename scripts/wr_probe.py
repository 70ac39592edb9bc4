"""HBM write-only bandwidth on an n x n complex128 buffer: cudaMemsetAsync
(torch zero_) and a fill (torch fill_), CUDA events; bytes written / time."""
import sys
import torch
n = int(sys.argv[1]) if len(sys.argv) > 1 else 81920
A = torch.empty(n * n, dtype=torch.complex128, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for label, fn in (("memset", lambda: A.zero_()), ("fill", lambda: A.fill_(1.0 + 2.0j))):
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(3):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{label}: {ms:.2f} ms, {16.0 * n * n / ms / 1e6:.0f} GB/s write")
