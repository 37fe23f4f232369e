"""Multi-GPU SymmSpMV: contiguous row blocks + a one-directional halo.

SURVEY §8(e) / DESIGN.md §8: the BFS-ordered rows are split into contiguous
blocks of whole tiles (balanced by nonzeros, `race_schedule_partition`).
Every stored entry points forward (col >= row), so rank p
  * needs x only from later ranks: x[R_{p+1} : halo_end_p)  (before the run),
  * produces y contributions for those same later rows      (after the run),
which are sent to their owners and added (in ascending sender order, so the
reduction order is fixed).  The exchange uses torch.distributed point-to-point
operations (NCCL over NVLink/NVSwitch on GPUs; gloo in the CPU tests and the
one-GPU multi-process test, staged through host memory): plumbing only; the
multiply and the halo add run in libsymmspmv.so kernels.

Overlap (SURVEY.md §8(e) "interior tiles run while C1 is in flight"): the
rank's plan splits its tiles into interior tiles (they touch own rows only)
and boundary tiles (they touch halo rows).  One multiply is
    post x-halo receives / sends            (NCCL stream)
    interior part: zero y, interior tiles   (compute stream, concurrently)
    wait for the x halo
    boundary part: boundary tiles
    y-halo send / receive, owner-side add kernel (ascending sender order).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def halo_pieces(bounds, halo_end, p):
    """[(q, a, b)]: rows [a, b) of rank p's halo that rank q > p owns."""
    out = []
    lo, hi = int(bounds[p + 1]), int(halo_end[p])
    for q in range(p + 1, len(bounds) - 1):
        a, b = max(lo, int(bounds[q])), min(hi, int(bounds[q + 1]))
        if a < b:
            out.append((q, a, b))
    return out


class HaloExchange:
    """Point-to-point halo plan of one rank (any torch.distributed backend;
    CUDA tensors are staged through host memory when the backend is not NCCL)."""

    def __init__(self, bounds, halo_end, rank: int, group=None):
        self.bounds = [int(v) for v in bounds]
        self.halo_end = [int(v) for v in halo_end]
        self.rank = rank
        self.group = group
        self.base = self.bounds[rank]
        # pieces of MY halo (owned by later ranks)
        self.mine = halo_pieces(self.bounds, self.halo_end, rank)
        # pieces of EARLIER ranks' halos that I own
        self.theirs = [(p, a, b) for p in range(rank) for (q, a, b) in halo_pieces(self.bounds, self.halo_end, p)
                       if q == rank]
        self.nccl = dist.get_backend(group) == "nccl"

    def _stage(self, t):
        """(tensor to hand to the backend, copy-back or None)."""
        if self.nccl or not t.is_cuda:
            return t, None
        h = t.detach().cpu()
        return h, (lambda: t.copy_(h))

    def post_x(self, x_loc: torch.Tensor):
        """x_loc covers [R_p, halo_end_p) with its own prefix filled: post the
        receives of the halo and the sends of the rows earlier ranks need.
        Returns a handle for wait_x (NCCL: the transfers run on NCCL's stream
        while the caller launches the interior part)."""
        b = self.base
        ops, backs = [], []
        for (q, a, c) in self.mine:
            t, back = self._stage(x_loc[a - b:c - b])
            ops.append(dist.P2POp(dist.irecv, t, q, self.group))
            if back:
                backs.append(back)
        for (p, a, c) in self.theirs:
            t, _ = self._stage(x_loc[a - b:c - b])
            ops.append(dist.P2POp(dist.isend, t, p, self.group))
        works = dist.batch_isend_irecv(ops) if ops else []
        return works, backs

    @staticmethod
    def wait_x(handle):
        works, backs = handle
        for w in works:
            w.wait()  # NCCL: the current stream waits for the transfer
        for back in backs:
            back()

    def exchange_x(self, x_loc: torch.Tensor):
        self.wait_x(self.post_x(x_loc))

    def reduce_y(self, y_loc: torch.Tensor, add):
        """Send my halo contributions to their owners; add the ones I receive
        into my own rows with `add(dst, buf)` (the C-ABI halo-add kernel on
        GPUs), in ascending sender rank order."""
        b = self.base
        bufs = [(a, torch.empty(c - a, dtype=y_loc.dtype, device=y_loc.device)) for (p, a, c) in self.theirs]
        ops, backs = [], []
        for (q, a, c) in self.mine:
            t, _ = self._stage(y_loc[a - b:c - b])
            ops.append(dist.P2POp(dist.isend, t, q, self.group))
        for (p, a, c), (_, buf) in zip(self.theirs, bufs):
            t, back = self._stage(buf)
            ops.append(dist.P2POp(dist.irecv, t, p, self.group))
            if back:
                backs.append(back)
        for w in (dist.batch_isend_irecv(ops) if ops else []):
            w.wait()
        for back in backs:
            back()
        for a, buf in bufs:  # ascending sender rank (self.theirs is ordered by p)
            add(y_loc[a - b:a - b + buf.numel()], buf)

    def halo_bytes(self) -> int:
        return 8 * sum(c - a for (_, a, c) in self.mine)


class DistSymmSpMV:
    """One rank of the multi-GPU SymmSpMV (tiled_atomic kernels on the rank's tiles)."""

    def __init__(self, sched, U=None, group=None, device: int | None = None, overlap: bool = True):
        import paper_1907_06487_b200 as P

        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)
        dev = torch.cuda.current_device() if device is None else device
        self.bounds, self.halo_end = sched.partition(self.nranks)
        self.plan = P.Plan(sched, U, variant="tiled_atomic", device=dev, nranks=self.nranks, rank=self.rank)
        self.hx = HaloExchange(self.bounds, self.halo_end, self.rank, group)
        self.row_begin, self.local_end = self.plan.local_range()
        self.own_end = int(self.bounds[self.rank + 1])
        self.overlap = overlap
        self._add = P.halo_add

    @property
    def n_own(self) -> int:
        return self.own_end - self.row_begin

    @property
    def n_local(self) -> int:
        return self.local_end - self.row_begin

    def parts(self) -> dict:
        return self.plan.parts()

    def empty_local(self):
        return torch.empty(self.n_local, dtype=torch.float64, device="cuda")

    def run(self, x_loc: torch.Tensor, y_loc: torch.Tensor):
        """x_loc, y_loc: CUDA float64 over [row_begin, local_end) (own rows first).
        On return y_loc[:n_own] holds this rank's rows of A x (permuted order)."""
        if self.overlap:
            h = self.hx.post_x(x_loc)                   # x halo in flight ...
            self.plan.run_part("interior", x_loc, y_loc)  # ... while the interior tiles run
            self.hx.wait_x(h)
            self.plan.run_part("boundary", x_loc, y_loc)
        else:
            self.hx.exchange_x(x_loc)
            self.plan.run(x_loc, y_loc)
        self.hx.reduce_y(y_loc, add=self._add)
