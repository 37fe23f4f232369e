"""Multi-GPU SymmSpMV: contiguous row blocks + a one-directional halo.

SURVEY §8(e) / DESIGN.md §8: the BFS-ordered rows are split into contiguous
blocks of whole tiles (balanced by nonzeros, `race_schedule_partition`).
Every stored entry points forward (col >= row), so rank p
  * needs x only from later ranks: x[R_{p+1} : halo_end_p)  (before the run),
  * produces y contributions for those same later rows      (after the run),
which are sent to their owners and added (in ascending sender order, so the
reduction order is fixed).  The exchange uses torch.distributed point-to-point
operations (NCCL over NVLink on GPUs, gloo in the CPU tests): plumbing only;
the multiply and the halo add run in libsymmspmv.so kernels.
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
    """Point-to-point halo plan of one rank (works for any torch.distributed backend)."""

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

    def _run(self, ops):
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    def exchange_x(self, x_loc: torch.Tensor):
        """x_loc covers [R_p, halo_end_p); its own prefix is filled; receive the halo."""
        b = self.base
        ops = [dist.P2POp(dist.irecv, x_loc[a - b:c - b], q, self.group) for (q, a, c) in self.mine]
        ops += [dist.P2POp(dist.isend, x_loc[a - b:c - b], p, self.group) for (p, a, c) in self.theirs]
        self._run(ops)

    def reduce_y(self, y_loc: torch.Tensor, add=None):
        """Send my halo contributions to their owners; add the ones I receive
        (ascending sender rank) into my own rows."""
        b = self.base
        bufs = [(a, torch.empty(c - a, dtype=y_loc.dtype, device=y_loc.device)) for (p, a, c) in self.theirs]
        ops = [dist.P2POp(dist.isend, y_loc[a - b:c - b], q, self.group) for (q, a, c) in self.mine]
        ops += [dist.P2POp(dist.irecv, buf, p, self.group) for (p, a, c), (_, buf) in zip(self.theirs, bufs)]
        self._run(ops)
        for a, buf in bufs:
            dst = y_loc[a - b:a - b + buf.numel()]
            if add is None:
                dst += buf
            else:
                add(dst, buf)

    def halo_bytes(self) -> int:
        return 8 * sum(c - a for (_, a, c) in self.mine)


class DistSymmSpMV:
    """One rank of the multi-GPU SymmSpMV (tiled_atomic kernels on the rank's tiles)."""

    def __init__(self, sched, U=None, group=None, device: int | None = None):
        import paper_1907_06487_b200 as P

        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)
        dev = torch.cuda.current_device() if device is None else device
        self.bounds, self.halo_end = sched.partition(self.nranks)
        self.plan = P.Plan(sched, U, variant="tiled_atomic", device=dev, nranks=self.nranks, rank=self.rank)
        self.hx = HaloExchange(self.bounds, self.halo_end, self.rank, group)
        self.row_begin, self.local_end = self.plan.local_range()
        self.own_end = int(self.bounds[self.rank + 1])
        self._add = P.halo_add

    @property
    def n_own(self) -> int:
        return self.own_end - self.row_begin

    @property
    def n_local(self) -> int:
        return self.local_end - self.row_begin

    def empty_local(self):
        return torch.empty(self.n_local, dtype=torch.float64, device="cuda")

    def run(self, x_loc: torch.Tensor, y_loc: torch.Tensor):
        """x_loc, y_loc: CUDA float64 over [row_begin, local_end) (own rows first).
        On return y_loc[:n_own] holds this rank's rows of A x (permuted order)."""
        self.hx.exchange_x(x_loc)
        self.plan.run(x_loc, y_loc)
        self.hx.reduce_y(y_loc, add=self._add)
