"""Multi-GPU drivers over torch.distributed (one process per GPU, NCCL over NVLink).

Two decompositions of the paper's R x C rank grid on one node:

* k-slab split (R = P, C = 1; primary).  Rank r owns the volume slab
  k in [kb[r], kb[r+1]) and the raw views [vb[r], vb[r+1]).  It filters its own
  views (Alg. alg:filter is row-separable), then one all-to-all sends to every
  rank h only the detector row band slab h projects onto (ifdk_band_rows), the
  NVLink analogue of the paper's per-projection MPI_Allgather cut
  down to the rows actually used.  Each rank then back-projects all views, in
  global view order, into its slab.  Slab starts are multiples of the kernel's
  64-slice chunk and view blocks are multiples of its 128-view summation batch,
  so the result is bitwise identical to one GPU.
* projection split (R = 1, C = P; variant).  Rank r back-projects its views
  into a full-size partial volume; a reduce-scatter (sum) of the contiguous
  k-slabs replaces the paper's single MPI_Reduce.  Needs a full
  volume per GPU, so it does not fit config 5.

The compute callables default to libifdk (``ifdk_filter`` / ``ifdk_backproject``);
tests inject the fp64 oracle to check the exchange logic on CPU with gloo.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

KC = 64          # slab starts are multiples of the BP kernel k-chunk (32 or 64, backproject.cu)
VIEW_BATCH = 128  # two-level summation batch of the BP kernel (BPParams.vb)


def _split(n: int, parts: int, quantum: int) -> list[int]:
    """Boundaries 0 = b0 <= ... <= b_parts = n, near-equal, interior ones on multiples of
    ``quantum`` whenever n is large enough."""
    out = [0]
    for r in range(1, parts):
        x = round(r * n / parts / quantum) * quantum
        if n < parts * quantum:
            x = round(r * n / parts)
        out.append(min(max(x, out[-1]), n))
    out.append(n)
    return out


@dataclass(frozen=True)
class SlabPlan:
    """Which slab and which views rank r owns (k-slab split)."""

    world: int
    Nz: int
    Np: int

    @property
    def k_bounds(self) -> list[int]:
        return _split(self.Nz, self.world, KC)

    @property
    def v_bounds(self) -> list[int]:
        return _split(self.Np, self.world, VIEW_BATCH)

    def slab(self, r: int) -> tuple[int, int]:
        kb = self.k_bounds
        return kb[r], kb[r + 1] - kb[r]

    def views(self, r: int) -> tuple[int, int]:
        vb = self.v_bounds
        return vb[r], vb[r + 1] - vb[r]


def band_union(g, k0: int, nk: int, s0: int, n: int) -> tuple[int, int]:
    """Union over views s0..s0+n-1 of the rows slab k0..k0+nk-1 needs (ifdk_band_rows)."""
    lo, hi = 1 << 30, -1
    for s in range(s0, s0 + n):
        a, b = g.band_rows(k0, nk, s)
        if a <= b:
            lo, hi = min(lo, a), max(hi, b)
    if hi < lo:
        return 0, -1
    return lo, hi


@dataclass
class Exchange:
    """Row bands of one all-to-all: send[h] = (lo, hi) of my views for slab h;
    recv[r] = (lo, hi) of rank r's views for my slab."""

    send: list[tuple[int, int]]
    recv: list[tuple[int, int]]


def plan_exchange(g, plan: SlabPlan, rank: int) -> Exchange:
    s0, n = plan.views(rank)
    send = []
    for h in range(plan.world):
        k0, nk = plan.slab(h)
        send.append(band_union(g, k0, nk, s0, n) if nk > 0 and n > 0 else (0, -1))
    k0, nk = plan.slab(rank)
    recv = []
    for r in range(plan.world):
        rs0, rn = plan.views(r)
        recv.append(band_union(g, k0, nk, rs0, rn) if nk > 0 and rn > 0 else (0, -1))
    return Exchange(send, recv)


def _rows(b):
    return max(b[1] - b[0] + 1, 0)


def kslab_reconstruct(g, raw_local, vol_slab, plan: SlabPlan, rank: int, group=None,
                      filter_fn: Optional[Callable] = None, bp_fn: Optional[Callable] = None,
                      timings: Optional[dict] = None):
    """k-slab FDK on one rank.  raw_local: [n_local][Nv][Nu] (views plan.views(rank));
    vol_slab: [nk][Ny][Nx] (slab plan.slab(rank)), overwritten."""
    import torch
    import torch.distributed as dist

    if filter_fn is None or bp_fn is None:
        from .ifdk import ifdk_backproject, ifdk_filter

        filter_fn = filter_fn or (lambda raw, out: ifdk_filter(g, raw, out))
        bp_fn = bp_fn or (lambda Q, s0, vol, k0, v0, acc: ifdk_backproject(
            g, Q, s0, vol, k0=k0, v0=v0, accumulate=acc))
    ev = (lambda: torch.cuda.Event(enable_timing=True)) if raw_local.is_cuda else None
    marks = [ev() for _ in range(4)] if (ev and timings is not None) else None
    if marks:
        marks[0].record()
    Q = torch.empty_like(raw_local)
    if raw_local.shape[0] > 0:
        filter_fn(raw_local, Q)
    if marks:
        marks[1].record()
    ex = plan_exchange(g, plan, rank)
    n_local = raw_local.shape[0]
    Nu = g.Nu
    recv_sizes = [plan.views(r)[1] * _rows(ex.recv[r]) * Nu for r in range(plan.world)]
    send_sizes = [n_local * _rows(b) * Nu for b in ex.send]
    if plan.world > 1:
        send_parts = [Q[:, lo:hi + 1, :].reshape(-1) for (lo, hi) in ex.send]
        send_buf = torch.cat(send_parts) if sum(send_sizes) else Q.new_empty(0)
        recv_buf = Q.new_empty(sum(recv_sizes))
        dist.all_to_all_single(recv_buf, send_buf, recv_sizes, send_sizes, group=group)
        del send_buf
    else:  # one rank: the band is read in place
        lo, hi = ex.recv[0]
        recv_buf = Q[:, lo:hi + 1, :].contiguous().reshape(-1) if _rows(ex.recv[0]) else Q.new_empty(0)
    if marks:
        marks[2].record()
    k0, nk = plan.slab(rank)
    off = 0
    first = True
    for r in range(plan.world):
        rs0, rn = plan.views(r)
        lo, hi = ex.recv[r]
        sz = recv_sizes[r]
        if rn > 0 and sz > 0 and nk > 0:
            band = recv_buf[off:off + sz].view(rn, hi - lo + 1, Nu)
            bp_fn(band, rs0, vol_slab, k0, lo, not first)
            first = False
        off += sz
    if first and nk > 0:
        vol_slab.zero_()
    if marks:
        marks[3].record()
        marks[3].synchronize()
        timings["filter_ms"] = marks[0].elapsed_time(marks[1])
        timings["exchange_ms"] = marks[1].elapsed_time(marks[2])
        timings["bp_ms"] = marks[2].elapsed_time(marks[3])
        timings["exchange_bytes_sent"] = 4 * sum(s for h, s in enumerate(send_sizes) if h != rank)
    return vol_slab


def projection_split_reconstruct(g, raw_local, s0: int, vol_slab, world: int, group=None,
                                 filter_fn: Optional[Callable] = None,
                                 bp_fn: Optional[Callable] = None):
    """Projection split: full partial volume per rank, then reduce-scatter (sum) of equal
    contiguous k-slabs (Nz must be divisible by world).  vol_slab: [Nz/world][Ny][Nx]."""
    import torch
    import torch.distributed as dist

    if filter_fn is None or bp_fn is None:
        from .ifdk import ifdk_backproject, ifdk_filter

        filter_fn = filter_fn or (lambda raw, out: ifdk_filter(g, raw, out))
        bp_fn = bp_fn or (lambda Q, s0_, vol, k0, v0, acc: ifdk_backproject(
            g, Q, s0_, vol, k0=k0, v0=v0, accumulate=acc))
    if g.Nz % world:
        raise ValueError("projection split needs Nz divisible by the world size")
    Q = torch.empty_like(raw_local)
    full = raw_local.new_empty((g.Nz, g.Ny, g.Nx))
    if raw_local.shape[0] > 0:
        filter_fn(raw_local, Q)
        bp_fn(Q, s0, full, 0, 0, False)
    else:
        full.zero_()
    if world > 1:
        dist.reduce_scatter_tensor(vol_slab, full, op=dist.ReduceOp.SUM, group=group)
    else:
        vol_slab.copy_(full)
    return vol_slab
