"""Row-slab sharding of the dense operator across GPUs.

One process per GPU (``torch.distributed``, NCCL on B200s).  Rank r owns rows
``[r0, r1)`` of A: its plan is built on the row slab of the test side
(``AssemblyPlan(..., row_begin=r0, row_end=r1)``, C++ ``row_slab``: the
elements touching those dofs, the other dofs constrained), while the trial
side is replicated, so the assembly needs no exchange at all.

The stored matvec is then ``y_r = A_r x`` on every rank with x replicated —
again no exchange.  Only a caller that needs the whole y on every rank (an
iterative solver building its Krylov basis) gathers the slabs: one all-gather
of 16 N bytes (1.3 MB for cfg 4), which is the only collective on this path.

The slabs are computed non-symmetrically (a rank cannot use G(x, y) = G(y, x)
across a slab boundary without writing into another rank's rows), so N ranks
do the work of N/2 single-GPU symmetric assemblies; the bench's multi-GPU mode
therefore stays "replicas".
"""
from __future__ import annotations

import torch

from . import AssemblyPlan, matvec as _matvec


def row_partition(n: int, world: int) -> list[tuple[int, int]]:
    """Contiguous row ranges, one per rank, sizes differing by at most one.

    Every row costs the same (a full row of trial locations), so equal row
    counts balance the assembly and the matvec."""
    if world < 1:
        raise ValueError("row_partition: world must be >= 1")
    base, extra = divmod(n, world)
    out, r0 = [], 0
    for r in range(world):
        r1 = r0 + base + (1 if r < extra else 0)
        out.append((r0, r1))
        r0 = r1
    return out


def _dist(group=None):
    """(dist, rank, world) of `group` (default: the whole job)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist, dist.get_rank(group), dist.get_world_size(group)
    return None, 0, 1


def gather_rows(y_local: torch.Tensor, n: int, group=None) -> torch.Tensor:
    """All ranks' row slabs of a vector (``row_partition`` order) -> the whole vector on every rank.

    Slabs are padded to the largest slab so that one ``all_gather_into_tensor``
    (NCCL) or ``all_gather`` (gloo) moves them; complex data travels as its
    real view."""
    dist, rank, world = _dist(group)
    parts = row_partition(n, world)
    if world == 1:
        return y_local
    width = max(r1 - r0 for r0, r1 in parts)
    real = torch.view_as_real(y_local) if y_local.is_complex() else y_local
    pad = torch.zeros((width,) + tuple(real.shape[1:]), dtype=real.dtype, device=real.device)
    pad[: real.shape[0]] = real
    if dist.get_backend(group) == "nccl":
        flat = torch.empty((world * width,) + tuple(real.shape[1:]), dtype=real.dtype, device=real.device)
        dist.all_gather_into_tensor(flat, pad, group=group)
        chunks = list(flat.split(width))
    else:
        chunks = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(chunks, pad, group=group)
    out = torch.cat([c[: r1 - r0] for c, (r0, r1) in zip(chunks, parts)])
    return torch.view_as_complex(out) if y_local.is_complex() else out


class ShardedOperator:
    """This rank's row slab of the dense single-layer operator, resident on its GPU.

    ``A`` is the (r1 - r0) x cols slab, column-major (``lda = max(1, r1 - r0)``),
    the same layout ``bem_dense`` returns for the whole matrix.  Rank and
    slab come from ``group`` (the whole job by default), and every device call
    runs with ``device`` current, so the plan's tables, the slab and the
    launches all live on that GPU."""

    def __init__(self, dom_x, dom_y, test, kernel, trial, opts=None, device=None, group=None):
        _, rank, world = _dist(group)
        self.rows = test.free_count()
        self.cols = trial.free_count()
        self.r0, self.r1 = row_partition(self.rows, world)[rank]
        self.group = group
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        args = (dom_x, dom_y, test, kernel, trial) + ((opts,) if opts is not None else ())
        with torch.cuda.device(self.device):
            self.plan = AssemblyPlan(*args, row_begin=self.r0, row_end=self.r1)
        self.lda = max(1, self.r1 - self.r0)
        self.A = torch.empty(self.cols * self.lda, dtype=torch.complex128, device=self.device)

    def assemble(self, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        if self.r1 > self.r0:
            with torch.cuda.device(self.device):
                self.plan.assemble(self.A.data_ptr(), self.lda, s.cuda_stream)
        return self

    def matvec_local(self, x: torch.Tensor, stream=None) -> torch.Tensor:
        """y[r0:r1] = A[r0:r1, :] x (x replicated, on this rank's device)."""
        if x.device != self.device:
            raise ValueError(f"ShardedOperator.matvec_local: x is on {x.device}, the slab on {self.device}")
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        y = torch.empty(self.r1 - self.r0, dtype=torch.complex128, device=self.device)
        if self.r1 > self.r0:
            with torch.cuda.device(self.device):
                _matvec(self.A.data_ptr(), self.r1 - self.r0, self.cols, self.lda, x.data_ptr(), y.data_ptr(),
                        s.cuda_stream)
        return y

    def matvec(self, x: torch.Tensor, stream=None) -> torch.Tensor:
        """The whole y = A x on every rank: local slab product + one all-gather."""
        return gather_rows(self.matvec_local(x, stream), self.rows, self.group)
