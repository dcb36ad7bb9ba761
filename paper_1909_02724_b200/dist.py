"""Multi-GPU drivers over torch.distributed (one process per GPU, NCCL over NVLink).

Two decompositions of the paper's R x C rank grid on one node:

* k-slab split (R = P, C = 1; primary).  Rank r owns the volume slab
  k in [kb[r], kb[r+1]) (slab starts are multiples of the BP kernel's 64-slice chunk).
  Views are sharded for filtering in blocks of ``block`` views, dealt round-robin:
  rank r owns blocks r, r + P, r + 2P, ...  Round t processes blocks tP .. tP+P-1, one
  per rank, i.e. the consecutive global views tPB .. (t+1)PB-1:
    filter (own block) -> pack the row band every slab needs (ifdk_band_rows)
    -> one all-to-all of the bands (the NVLink analogue of the paper's per-projection
       MPI_Allgather, cut down to the rows actually used)
    -> back-project the P received blocks, in global view order, into the own slab.
  Rounds are software-pipelined on CUDA streams (the paper's filter / exchange / BP
  threads, as streams): filter + exchange of round t+1 overlap the
  back-projection of round t.  Because blocks are multiples of the kernel's 128-view
  summation batch and arrive in global order, every slab is bitwise identical to one GPU.
* projection split (R = 1, C = P; variant).  Rank r back-projects its views
  into a full-size partial volume; a reduce-scatter (sum) of the contiguous
  k-slabs replaces the paper's single MPI_Reduce.  Needs a full
  volume per GPU, so it does not fit config 5.
* fused projection split (``projection_split_fused``): the same decomposition with the
  reduce inside the back-projection's write-back -- every 128-view partial sum is added
  (``ifdk_backproject_reduce``: red.global.add over NVLink, or multimem.red on multicast
  mappings) straight into the owner's slab, mapped into every rank (``ReduceSlabs``, CUDA
  IPC).  No partial volume and no reduce-scatter: a rank holds its filtered views and its own
  slab only, so config 5 fits.

The band exchange is fused into the filter by default: ``PeerExchange`` maps every rank's
receive buffer into every other rank (CUDA IPC over NVLink), ``ifdk_filter_scatter`` stores
each filtered row straight into the destination bands, and device-side signals
(``ifdk_signal`` / ``ifdk_wait``) order the stores before the peers' back-projection and
the buffer reuse after it.  NCCL ``all_to_all_single`` is the baseline (``exchange="nccl"``).

``kslab_reconstruct_host`` is the end-to-end form: raw blocks come from pinned host
memory (H2D on a copy stream, one round ahead) and the finished slab goes back to the
host in sub-slabs while the last round's back-projection continues.

The compute callables default to libifdk (``ifdk_filter`` / ``ifdk_backproject``);
tests inject the fp64 oracle to check the exchange logic on CPU with gloo.
"""
from __future__ import annotations

import contextlib
from dataclasses import dataclass, field
from typing import Callable, Optional

KC = 64          # slab starts are multiples of the BP kernel k-chunk (32 or 64, backproject.cu)
VIEW_BATCH = 128  # two-level summation batch of the BP kernel (BPParams.vb)
D2H_SUBSLAB = 256  # slices per device-to-host piece of the end-to-end driver (multiple of KC)
D2H_TAIL = 64      # ... and per piece of the slab's last 256 slices (the D2H nothing overlaps)


def _d2h_pieces(k0: int, nk: int) -> list:
    """(first slice, slices) pieces of slab k0..k0+nk-1 for the streamed D2H of the last
    round: D2H_SUBSLAB-slice pieces, the last D2H_SUBSLAB slices in D2H_TAIL-slice ones
    (all boundaries stay multiples of 64 relative to k0, so the result is unchanged)."""
    out, a, end = [], k0, k0 + nk
    while a + 2 * D2H_SUBSLAB <= end:
        out.append((a, D2H_SUBSLAB))
        a += D2H_SUBSLAB
    while a < end:
        out.append((a, min(D2H_TAIL, end - a)))
        a += D2H_TAIL
    return out


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
    """Which slab rank r owns, and which view blocks (k-slab split).

    The plan covers the global view blocks offset, offset + stride, offset + 2 stride, ...
    (all blocks by default; one column of an R x C grid otherwise, see hybrid_reconstruct)."""

    world: int
    Nz: int
    Np: int
    block: int = VIEW_BATCH
    stride: int = 1
    offset: int = 0

    @property
    def k_bounds(self) -> list[int]:
        return _split(self.Nz, self.world, KC)

    def slab(self, r: int) -> tuple[int, int]:
        kb = self.k_bounds
        return kb[r], kb[r + 1] - kb[r]

    @property
    def n_blocks(self) -> int:
        total = (self.Np + self.block - 1) // self.block
        return max(0, (total - self.offset + self.stride - 1) // self.stride)

    @property
    def n_rounds(self) -> int:
        return (self.n_blocks + self.world - 1) // self.world

    def block_views(self, b: int) -> tuple[int, int]:
        """(first global view, count) of the plan's block b (count 0 past the end)."""
        if b >= self.n_blocks:
            return self.Np, 0
        s0 = (self.offset + b * self.stride) * self.block
        return s0, max(0, min(self.block, self.Np - s0))

    def round_block(self, t: int, r: int) -> tuple[int, int]:
        """The block rank r filters in round t."""
        return self.block_views(t * self.world + r)

    def local_views(self, r: int) -> list[tuple[int, int]]:
        """Rank r's blocks (global first view, count) in local storage order."""
        return [self.round_block(t, r) for t in range(self.n_rounds)
                if self.round_block(t, r)[1] > 0]

    def n_local(self, r: int) -> int:
        return sum(n for _, n in self.local_views(r))


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


def _rows(b):
    return max(b[1] - b[0] + 1, 0)


@dataclass
class Exchange:
    """Row bands of one round's all-to-all: send[h] = (lo, hi) of my block for slab h;
    recv[r] = (lo, hi) of rank r's block for my slab; views[r] = (s0, n) of r's block."""

    send: list[tuple[int, int]]
    recv: list[tuple[int, int]]
    views: list[tuple[int, int]]
    send_sizes: list[int] = field(default_factory=list)
    recv_sizes: list[int] = field(default_factory=list)


_EXCHANGE_CACHE: dict = {}


def exchanges(g, plan: SlabPlan, rank: int) -> list[Exchange]:
    """plan_exchange for every round (cached per geometry, plan and rank)."""
    key = (g.Nu, g.Nv, g.Nx, g.Ny, g.Nz, g.Du, g.Dv, g.Dx, g.Dy, g.Dz, g.D, g.d, g.theta,
           plan, rank)
    if key not in _EXCHANGE_CACHE:
        if len(_EXCHANGE_CACHE) > 64:
            _EXCHANGE_CACHE.clear()
        _EXCHANGE_CACHE[key] = [plan_exchange(g, plan, rank, t) for t in range(plan.n_rounds)]
    return _EXCHANGE_CACHE[key]


def plan_exchange(g, plan: SlabPlan, rank: int, t: int) -> Exchange:
    """The bands of round t as seen by ``rank`` (both directions)."""
    s0, n = plan.round_block(t, rank)
    send = []
    for h in range(plan.world):
        k0, nk = plan.slab(h)
        send.append(band_union(g, k0, nk, s0, n) if nk > 0 and n > 0 else (0, -1))
    k0, nk = plan.slab(rank)
    recv, views = [], []
    for r in range(plan.world):
        rs0, rn = plan.round_block(t, r)
        views.append((rs0, rn))
        recv.append(band_union(g, k0, nk, rs0, rn) if nk > 0 and rn > 0 else (0, -1))
    ex = Exchange(send, recv, views)
    ex.send_sizes = [n * _rows(b) * g.Nu for b in send]
    ex.recv_sizes = [views[r][1] * _rows(recv[r]) * g.Nu for r in range(plan.world)]
    return ex


class _Streams:
    """CUDA streams/events for the pipeline, or no-ops for CPU tensors (gloo tests)."""

    def __init__(self, cuda: bool, streams=None):
        import torch

        self.cuda = cuda
        self.torch = torch
        if cuda and streams is not None:
            self.F, self.B, self.C = streams
        elif cuda:
            self.F = torch.cuda.Stream()  # filter + band packing (+ exchange issue)
            self.B = torch.cuda.Stream()  # back-projection
            self.C = torch.cuda.Stream()  # host copies
        else:
            self.F = self.B = self.C = None

    def on(self, s):
        return self.torch.cuda.stream(s) if self.cuda else contextlib.nullcontext()

    def event(self, timing=False):
        return self.torch.cuda.Event(enable_timing=timing) if self.cuda else None

    def record(self, ev, s):
        if ev is not None:
            ev.record(s)

    def wait(self, s, ev):
        if ev is not None and s is not None:
            s.wait_event(ev)


def _default_fns(g, filter_fn, bp_fn):
    if filter_fn is None or bp_fn is None:
        from .ifdk import ifdk_backproject, ifdk_filter

        filter_fn = filter_fn or (lambda raw, out: ifdk_filter(g, raw, out))
        bp_fn = bp_fn or (lambda Q, s0, vol, k0, v0, acc: ifdk_backproject(
            g, Q, s0, vol, k0=k0, v0=v0, accumulate=acc))
    return filter_fn, bp_fn


class PeerExchange:
    """Receive buffers of the fused row-band exchange, one per rank and mapped into every rank
    (CUDA IPC: NVLink peer memory between GPUs), plus the signal words that order the peers'
    stores (ifdk_filter_scatter's completion flags, ifdk_signal / ifdk_wait; the ordering
    argument is in csrc/peer.cu).

    Layout of rank h's buffer (bytes): [0, 256) uint32 landed[r] = rounds of rank r's rows
    that have landed in h's receive area; [256, 512) uint32 freed[r] = rounds rank r has
    back-projected (buffer releases); [512, 516) the ticket of h's own scatter launches;
    [1024, ...) the fp32 receive area, two rounds deep: 2 * recv_max[h] floats.  Every rank
    signals every other rank once per round (rows or not), so after round t every landed[r]
    is t + 1 and, once its back-projection is done, every freed[r] is t + 1.

    ``create`` builds one over a process group (IPC handles exchanged with all_gather_object);
    ``local`` builds all ranks' exchanges in one process on one GPU (virtual ranks, tests)."""

    HEADER = 1024

    def __init__(self, rank, world, bases, recv_max, own=(), opened=()):
        if world > 16:
            raise ValueError("the fused exchange signals at most 16 ranks")
        self.rank, self.world = rank, world
        self.bases = [int(b) for b in bases]
        self.recv_max = list(recv_max)
        self._own, self._opened = list(own), list(opened)
        self.kind = "p2p-fused"
        # rounds of earlier pipeline calls: the signal words count on from there (every rank
        # runs the same calls with the same number of rounds)
        self.rounds_done = 0
        self.timeout_ms = 0  # of the wait kernels (0: the library's 300 s)

    # -- construction
    @staticmethod
    def _alloc(recv_max):
        from .ifdk import as_tensor, peer_alloc

        ptr, handle = peer_alloc(PeerExchange.HEADER + 8 * max(int(recv_max), 1))
        as_tensor(ptr, (PeerExchange.HEADER // 4,), "uint32").zero_()
        return ptr, handle

    @classmethod
    def create(cls, group, rank, world, recv_max):
        import torch
        import torch.distributed as dist

        from .ifdk import peer_open

        ptr, handle = cls._alloc(recv_max[rank])
        handles = [None] * world
        dist.all_gather_object(handles, handle, group=group)
        bases, opened = [], []
        for h in range(world):
            if h == rank:
                bases.append(ptr)
            else:
                q = peer_open(handles[h])
                bases.append(q)
                opened.append(q)
        torch.cuda.synchronize()
        dist.barrier(group=group)  # every header zeroed before anyone signals
        return cls(rank, world, bases, recv_max, own=[ptr], opened=opened)

    @classmethod
    def local(cls, world, recv_max):
        ptrs = [cls._alloc(recv_max[h])[0] for h in range(world)]
        ex = [cls(r, world, ptrs, recv_max) for r in range(world)]
        ex[0]._own = ptrs  # rank 0's object frees them all
        return ex

    def close(self):
        from .ifdk import peer_close, peer_free

        for q in self._opened:
            peer_close(q)
        for q in self._own:
            peer_free(q)
        self._opened, self._own = [], []

    # -- addressing
    def _area(self, h, q, off):
        return self.bases[h] + self.HEADER + 4 * (q * self.recv_max[h] + off)

    def recv(self, q, off, rn, rows, Nu):
        """My receive area q at element offset off as a [rn][rows][Nu] tensor."""
        from .ifdk import as_tensor

        return as_tensor(self._area(self.rank, q, off), (rn, rows, Nu))

    def _landed_flags(self):
        return [b + 4 * self.rank for b in self.bases]

    # -- the round protocol (each call enqueues on the current stream)
    def wait_free(self, t):
        """Before scattering round t: every rank has released buffer t % 2 (round t - 2 of
        this call, or every round of the earlier calls)."""
        from .ifdk import ifdk_wait

        target = self.rounds_done + (t - 1 if t >= 2 else 0)
        if target > 0:
            ifdk_wait(self.bases[self.rank] + 256, self.world, target, self.timeout_ms)

    def scatter(self, g, src, q, bands, filter_fn=None):
        """Filter src (the rank's block of this round, None if it has none) into every
        destination band: bands = [(h, off, lo, hi)] (element offset off in h's receive
        layout); raises every rank's landed word once all rows have been stored.  The filter
        is ifdk_filter_scatter's (bitwise ifdk_filter's); filter_fn is for host fakes."""
        from .ifdk import ifdk_filter_scatter, ifdk_signal

        dests = [(self._area(h, q, off), lo, hi) for h, off, lo, hi in bands]
        if src is not None and dests:
            ifdk_filter_scatter(g, src, dests, flags=self._landed_flags(),
                                ticket=self.bases[self.rank] + 512)
        else:
            ifdk_signal(self._landed_flags())

    def wait_landed(self, t):
        from .ifdk import ifdk_wait

        ifdk_wait(self.bases[self.rank], self.world, self.rounds_done + t + 1, self.timeout_ms)

    def release(self):
        """After back-projecting a round: tell every rank its buffer here may be reused."""
        from .ifdk import ifdk_signal

        ifdk_signal([b + 256 + 4 * self.rank for b in self.bases])


_P2P_CACHE: dict = {}


def _peer_exchange(group, rank, world, recv_max, dev):
    """A PeerExchange over `group` (cached: creation is collective and the buffers persist),
    or None on every rank if any rank cannot map its peers."""
    import torch
    import torch.distributed as dist

    key = (id(group or dist.group.WORLD), rank, world, tuple(recv_max), str(dev))
    if key in _P2P_CACHE:
        return _P2P_CACHE[key]
    ex, err = None, None
    try:
        ex = PeerExchange.create(group, rank, world, recv_max)
    except Exception as exc:  # noqa: BLE001 -- no peer mapping: the NCCL band exchange
        err = exc
    on_dev = dist.get_backend(group) == "nccl"
    ok = torch.tensor([1 if ex is not None else 0], device=dev if on_dev else "cpu")
    dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
    if int(ok.item()) == 0:
        import warnings

        warnings.warn(f"peer memory unavailable, NCCL band exchange: {err!r}")
        if ex is not None:
            ex.close()
        ex = None
    if ex is not None:
        if len(_P2P_CACHE) > 4:
            for old in _P2P_CACHE.values():
                if old is not None:
                    old.close()
            _P2P_CACHE.clear()
        _P2P_CACHE[key] = ex
    return ex


def _pipeline(g, plan: SlabPlan, rank: int, vol_slab, group, filter_fn, bp_fn, timings,
              raw_local=None, raw_host=None, vol_host=None, force_exchange=False,
              exchange="auto", peer=None, streams=None):
    import torch
    import torch.distributed as dist

    filter_fn, bp_fn = _default_fns(g, filter_fn, bp_fn)
    world = plan.world
    # exchange through the process group even at world size 1 (exercises the collective on
    # the pipeline's streams; the band is then packed and "sent" to itself)
    xchg = world > 1 or (force_exchange and dist.is_available() and dist.is_initialized())
    k0, nk = plan.slab(rank)
    # vol_slab None: bp_fn writes elsewhere (the fused reduce of hybrid_reconstruct) and is
    # called with vol None; slices no view touches are then left as they are
    src = vol_slab if vol_slab is not None else (raw_local if raw_local is not None else raw_host)
    cuda = src.is_cuda or (vol_slab is None and torch.cuda.is_available() and raw_host is not None)
    S = _Streams(cuda, streams)
    dev = src.device if src.is_cuda or vol_slab is not None else torch.device("cuda")
    Nv, Nu = g.Nv, g.Nu
    rounds = plan.n_rounds
    exs = exchanges(g, plan, rank)
    my_blocks = plan.local_views(rank)
    offs, o = [], 0
    for _, n in my_blocks:
        offs.append(o)
        o += n
    B = plan.block
    send_max = max([sum(e.send_sizes) for e in exs] + [1])
    # receive-area size of every rank (the fused exchange addresses the destination's layout)
    recv_max_all = [max([sum(e.recv_sizes) for e in exchanges(g, plan, h)] + [1])
                    for h in range(world)]
    recv_max = recv_max_all[rank]
    if peer is None and xchg and cuda and exchange in ("auto", "p2p"):
        peer = _peer_exchange(group, rank, world, recv_max_all, dev)
        if peer is None and exchange == "p2p":
            raise RuntimeError("exchange='p2p': peer memory unavailable")
    if not xchg:
        peer = None
    if peer is not None and cuda:
        # the one torch kernel the pipeline may launch (zero_ of untouched slices), loaded now:
        # under lazy module loading a first launch behind a spinning wait kernel would
        # deadlock (csrc/peer.cu preloads the library's own kernels the same way)
        torch.zeros(1, device=dev)
    nbuf = min(2, rounds)
    if peer is not None:
        Qbuf = [None] * nbuf
        sendbuf = recvbuf = None
        # element offset of my band inside destination h's receive layout, per round
        p2p_off = [[sum(exchanges(g, plan, h)[t].recv_sizes[:rank]) for h in range(world)]
                   for t in range(rounds)]
    else:
        # Persistent double buffers (no allocator traffic across streams).
        Qbuf = [torch.empty((B, Nv, Nu), device=dev) for _ in range(nbuf)]
        sendbuf = [torch.empty(send_max, device=dev) for _ in Qbuf] if xchg else None
        recvbuf = [torch.empty(recv_max, device=dev) for _ in Qbuf] if xchg else None
    stage = [torch.empty((B, Nv, Nu), device=dev) for _ in Qbuf] if raw_host is not None else None

    cur = torch.cuda.current_stream() if cuda else None
    t_start = S.event(True)
    S.record(t_start, cur)
    for s in (S.F, S.B, S.C):
        S.wait(s, t_start)
    ev_bp_done = [None, None]
    ev_filt_done = [None, None]
    ev_h2d = [None, None]
    f_marks, b_marks, c_marks = [], [], []

    def h2d(t):  # round t's own raw block -> stage[t % 2] on the copy stream
        if raw_host is None or t >= rounds or plan.round_block(t, rank)[1] == 0:
            return
        q = t % 2
        n = plan.round_block(t, rank)[1]
        bi = sum(1 for tt in range(t) if plan.round_block(tt, rank)[1] > 0)
        with S.on(S.C):
            S.wait(S.C, ev_filt_done[q])  # stage[q] free once filter(t-2) has read it
            e0 = S.event(True)
            S.record(e0, S.C)
            stage[q][:n].copy_(raw_host[offs[bi]:offs[bi] + n], non_blocking=True)
            ev_h2d[q] = S.event(True)
            S.record(ev_h2d[q], S.C)
            c_marks.append((e0, ev_h2d[q]))

    h2d(0)
    first_bp = True
    bi = 0
    for t in range(rounds):
        q = t % 2
        ex = exs[t]
        s0, n = plan.round_block(t, rank)
        h2d(t + 1)
        with S.on(S.F):
            # sendbuf[q] / recvbuf[q] / Qbuf[q] were last used by round t-2's BP
            S.wait(S.F, ev_bp_done[q])
            e0 = S.event(True)
            S.record(e0, S.F)
            src = None
            if n > 0:
                if raw_host is not None:
                    S.wait(S.F, ev_h2d[q])
                    src = stage[q][:n]
                else:
                    src = raw_local[offs[bi]:offs[bi] + n]
            work = None
            if peer is not None:
                # fused: every filtered row goes straight into the receive areas of the slabs
                # that need it (NVLink stores into peer memory).  Before: every rank has
                # released area q (its BP of round t - 2 is done); after the last store the
                # kernel raises this rank's landed word on every rank (csrc/peer.cu).
                peer.wait_free(t)
                bands = [(h, p2p_off[t][h], lo, hi) for h, (lo, hi) in enumerate(ex.send)
                         if hi >= lo]
                peer.scatter(g, src if n > 0 else None, q, bands, filter_fn)
                if n > 0:
                    bi += 1
                e1 = S.event(True)
                S.record(e1, S.F)
                f_marks.append((e0, e1))
            elif xchg:
                if n > 0:
                    filter_fn(src, Qbuf[q][:n])
                    bi += 1
                    off = 0
                    for (lo, hi), sz in zip(ex.send, ex.send_sizes):
                        if sz:
                            sendbuf[q][off:off + sz].view(n, hi - lo + 1, Nu).copy_(
                                Qbuf[q][:n, lo:hi + 1, :])
                        off += sz
                e1 = S.event(True)
                S.record(e1, S.F)
                f_marks.append((e0, e1))
                work = dist.all_to_all_single(recvbuf[q][:sum(ex.recv_sizes)],
                                              sendbuf[q][:sum(ex.send_sizes)],
                                              ex.recv_sizes, ex.send_sizes, group=group,
                                              async_op=True)
            else:
                if n > 0:
                    filter_fn(src, Qbuf[q][:n])
                    bi += 1
                e1 = S.event(True)
                S.record(e1, S.F)
                f_marks.append((e0, e1))
            ev_filt_done[q] = S.event()  # stage[q] may be refilled
            S.record(ev_filt_done[q], S.F)
            ev_ready = S.event()
            S.record(ev_ready, S.F)
        with S.on(S.B):
            if work is not None:
                work.wait()  # the BP stream waits for the collective
            S.wait(S.B, ev_ready)
            if peer is not None:
                peer.wait_landed(t)  # every rank's round-t rows are in my area q
            b0 = S.event(True)
            S.record(b0, S.B)
            last = t == rounds - 1
            # the last round goes in sub-slabs so that finished slices leave for the host early
            subs = [(k0, nk)]
            if last and vol_host is not None and nk > D2H_TAIL:
                subs = _d2h_pieces(k0, nk)
            launched = False
            for (a, m) in subs:
                acc_first = first_bp
                off = 0
                for r in range(world):
                    rs0, rn = ex.views[r]
                    lo, hi = ex.recv[r]
                    sz = ex.recv_sizes[r]
                    if rn > 0 and sz > 0 and nk > 0:
                        if peer is not None:
                            band, v0 = peer.recv(q, off, rn, hi - lo + 1, Nu), lo
                        elif xchg:
                            band, v0 = recvbuf[q][off:off + sz].view(rn, hi - lo + 1, Nu), lo
                        else:  # one rank: back-project straight from the filtered block
                            band, v0 = Qbuf[q][:rn], 0
                        bp_fn(band, rs0, None if vol_slab is None else vol_slab[a - k0:a - k0 + m],
                              a, v0, not acc_first)
                        acc_first = False
                        launched = True
                    off += sz
                if last and acc_first and vol_slab is not None:  # no view touches these slices
                    vol_slab[a - k0:a - k0 + m].zero_()
                if last and vol_host is not None and m > 0:
                    ev = S.event()
                    S.record(ev, S.B)
                    with S.on(S.C):
                        S.wait(S.C, ev)
                        c0 = S.event(True)
                        S.record(c0, S.C)
                        vol_host[a - k0:a - k0 + m].copy_(vol_slab[a - k0:a - k0 + m],
                                                          non_blocking=True)
                        c1 = S.event(True)
                        S.record(c1, S.C)
                        c_marks.append((c0, c1))
            if peer is not None:
                peer.release()  # my area q may be refilled (round t + 2)
            if launched:
                first_bp = False
            b1 = S.event(True)
            S.record(b1, S.B)
            b_marks.append((b0, b1))
            ev_bp_done[q] = S.event()
            S.record(ev_bp_done[q], S.B)
    if peer is not None:
        peer.rounds_done += rounds
    if rounds == 0 and nk > 0 and vol_slab is not None:  # no views at all
        vol_slab.zero_()
        if vol_host is not None:
            vol_host.copy_(vol_slab)
    if cuda:
        for s in (S.F, S.B, S.C):
            cur.wait_stream(s)
    t_end = S.event(True)
    S.record(t_end, cur)
    if timings is not None and cuda:
        t_end.synchronize()
        wall = t_start.elapsed_time(t_end)
        tf = sum(a.elapsed_time(b) for a, b in f_marks)
        tb = sum(a.elapsed_time(b) for a, b in b_marks)
        tc = sum(a.elapsed_time(b) for a, b in c_marks)
        timings.update({"wall_ms": wall, "filter_pack_ms": tf, "bp_ms": tb, "host_copy_ms": tc,
                        "rounds": rounds,
                        "exchange": (peer.kind if peer is not None else "nccl") if xchg
                        else "none",
                        "delta": (tf + tb + tc) / wall if wall > 0 else None,
                        "exchange_bytes_sent": 4 * sum(sum(e.send_sizes) - e.send_sizes[rank]
                                                       for e in exs) if xchg else 0})
    return vol_slab


def kslab_reconstruct(g, raw_local, vol_slab, plan: SlabPlan, rank: int, group=None,
                      filter_fn: Optional[Callable] = None, bp_fn: Optional[Callable] = None,
                      timings: Optional[dict] = None, force_exchange: bool = False,
                      exchange: str = "auto", peer: Optional[PeerExchange] = None,
                      streams=None):
    """k-slab FDK on one rank.  raw_local: [plan.n_local(rank)][Nv][Nu], the rank's blocks
    (plan.local_views(rank)) in order, device-resident; vol_slab: [nk][Ny][Nx] (slab
    plan.slab(rank)), overwritten.  Enqueued on side streams that the current stream joins.
    exchange: "auto" fuses the band exchange into the filter over peer (NVLink) memory when
    every rank can map its peers (PeerExchange: ifdk_filter_scatter + device-side signals),
    else NCCL all-to-all; "p2p" requires the fused exchange; "nccl" forces the all-to-all.
    peer: an existing PeerExchange (e.g. PeerExchange.local for virtual ranks on one GPU);
    streams: (filter, back-projection, copy) streams to use instead of three new ones."""
    return _pipeline(g, plan, rank, vol_slab, group, filter_fn, bp_fn, timings,
                     raw_local=raw_local, force_exchange=force_exchange, exchange=exchange,
                     peer=peer, streams=streams)


def kslab_reconstruct_host(g, raw_host, vol_slab, vol_host, plan: SlabPlan, rank: int,
                           group=None, filter_fn: Optional[Callable] = None,
                           bp_fn: Optional[Callable] = None, timings: Optional[dict] = None,
                           force_exchange: bool = False, exchange: str = "auto",
                           peer: Optional[PeerExchange] = None, streams=None):
    """End-to-end k-slab FDK on one rank: raw_host (pinned, the rank's blocks in order) is
    copied block by block one round ahead; vol_slab (device scratch [nk][Ny][Nx]) is
    streamed to vol_host (pinned) in sub-slabs during the last round."""
    return _pipeline(g, plan, rank, vol_slab, group, filter_fn, bp_fn, timings,
                     raw_host=raw_host, vol_host=vol_host, force_exchange=force_exchange,
                     exchange=exchange, peer=peer, streams=streams)


# ------------------------------------------------------------------ fused projection split
class ReduceSlabs:
    """The owner slabs of the fused projection-split reduce, each mapped into every rank:
    rank h's slab (its device memory; CUDA IPC makes it an NVLink peer mapping elsewhere)
    holds slices k_bounds[h] .. k_bounds[h+1]-1 of the [Nz][Ny][Nx] volume.  ``create``
    builds them over a process group, ``local`` all of them in one process (virtual ranks)."""

    kind = "p2p-red"

    def __init__(self, rank, world, bases, k_bounds, Ny, Nx, own=(), opened=()):
        self.rank, self.world = rank, world
        self.bases = [int(b) for b in bases]
        self.k_bounds = list(k_bounds)
        self.Ny, self.Nx = Ny, Nx
        self._own, self._opened = list(own), list(opened)

    @staticmethod
    def _alloc(nk, Ny, Nx):
        from .ifdk import peer_alloc

        return peer_alloc(4 * max(nk, 1) * Ny * Nx)

    @classmethod
    def create(cls, group, rank, world, g, k_bounds):
        import torch.distributed as dist

        from .ifdk import peer_open

        ptr, handle = cls._alloc(k_bounds[rank + 1] - k_bounds[rank], g.Ny, g.Nx)
        handles = [None] * world
        dist.all_gather_object(handles, handle, group=group)
        bases, opened = [], []
        for h in range(world):
            if h == rank:
                bases.append(ptr)
            else:
                q = peer_open(handles[h])
                bases.append(q)
                opened.append(q)
        return cls(rank, world, bases, k_bounds, g.Ny, g.Nx, own=[ptr], opened=opened)

    @classmethod
    def local(cls, world, g, k_bounds):
        ptrs = [cls._alloc(k_bounds[h + 1] - k_bounds[h], g.Ny, g.Nx)[0] for h in range(world)]
        out = [cls(r, world, ptrs, k_bounds, g.Ny, g.Nx) for r in range(world)]
        out[0]._own = ptrs  # rank 0's object frees them all
        return out

    def dests(self):
        """(bases, first slices) of the non-empty slabs, for ifdk_backproject_reduce."""
        kb = self.k_bounds
        keep = [h for h in range(self.world) if kb[h + 1] > kb[h]]
        return [self.bases[h] for h in keep], [kb[h] for h in keep]

    def slab(self, h=None):
        """Slab h (default: my own) as a device tensor [nk][Ny][Nx] over its mapping."""
        from .ifdk import as_tensor

        h = self.rank if h is None else h
        return as_tensor(self.bases[h], (self.k_bounds[h + 1] - self.k_bounds[h], self.Ny, self.Nx))

    def close(self):
        from .ifdk import peer_close, peer_free

        for q in self._opened:
            peer_close(q)
        for q in self._own:
            peer_free(q)
        self._opened, self._own = [], []


def projection_split_fused(g, raw_local, blocks, slabs, group=None,
                           filter_fn: Optional[Callable] = None,
                           reduce_fn: Optional[Callable] = None,
                           timings: Optional[dict] = None, mode: int = 0, zero: bool = True,
                           sync: bool = True):
    """Fused projection split on one rank: filter the rank's views (``blocks``: (first global
    view, count) runs stored in raw_local, in order) and back-project them over the whole
    volume, each 128-view partial sum added straight into its owner's slab
    (``ifdk_backproject_reduce`` into ``slabs``, a ReduceSlabs).  zero / sync: zero the own
    slab and order it before every rank's adds, and order every rank's adds before the
    return (a device sync + a group barrier each); virtual ranks in one process pass False and
    order the calls themselves.  Returns the own slab (a tensor over its mapping).  Equal to
    one GPU up to fp32 summation order (the adds' order across ranks is not fixed)."""
    import torch

    from .ifdk import ifdk_backproject_reduce, ifdk_filter

    if filter_fn is None:
        def filter_fn(raw, out):
            ifdk_filter(g, raw, out)
    if reduce_fn is None:
        bases, k0s = slabs.dests()

        def reduce_fn(Qb, s0):
            ifdk_backproject_reduce(g, Qb, s0, bases, k0s, 0, g.Nz, mode=mode)
    barrier = _barrier_fn(group) if sync else (lambda: None)
    cuda = raw_local.is_cuda
    if zero:
        slabs.slab().zero_()
    if sync:
        if cuda:
            torch.cuda.synchronize()
        barrier()  # every slab zeroed before any rank adds into it
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)] if (cuda and timings is not None) else None
    if ev:
        ev[0].record()
    Q = torch.empty_like(raw_local)
    if raw_local.shape[0] > 0:
        filter_fn(raw_local, Q)
    if ev:
        ev[1].record()
    off = 0
    for s0, n in blocks:
        if n > 0:
            reduce_fn(Q[off:off + n], s0)
        off += n
    if ev:
        ev[2].record()
    if sync:
        if cuda:
            torch.cuda.synchronize()
        barrier()  # every rank's adds have landed
    if ev:
        ev[2].synchronize()
        timings.update({"filter_ms": ev[0].elapsed_time(ev[1]),
                        "bp_reduce_ms": ev[1].elapsed_time(ev[2]),
                        "wall_ms": ev[0].elapsed_time(ev[2])})
    del Q
    return slabs.slab()


def _barrier_fn(group):
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return lambda: None
    return lambda: dist.barrier(group=group)


# ----------------------------------------------------------------------------- R x C grid
@dataclass(frozen=True)
class GridPlan:
    """The paper's R x C rank grid: rank = r C + c.  Row r owns volume slab r of R
    (multiples of the 64-slice chunk); column c owns the view blocks b = c (mod C).  Inside a
    column the k-slab pipeline runs over its R ranks (band all-to-all); across a row the C
    partial slabs are summed by a reduce-scatter, leaving rank (r, c) the c-th of C equal
    sub-slabs of slab r.  R = P, C = 1 is the k-slab split; R = 1, C = P the projection split."""

    R: int
    C: int
    Nz: int
    Np: int
    block: int = VIEW_BATCH

    def coords(self, rank: int) -> tuple[int, int]:
        return rank // self.C, rank % self.C

    def column_plan(self, c: int) -> SlabPlan:
        return SlabPlan(self.R, self.Nz, self.Np, self.block, stride=self.C, offset=c)

    def slab(self, r: int) -> tuple[int, int]:
        return SlabPlan(self.R, self.Nz, self.Np).slab(r)

    def sub_bounds(self, r: int) -> list[int]:
        """Split of slab r into C sub-slabs (the fused row reduce's owner slabs; multiples of
        the 64-slice chunk where the slab is long enough): C + 1 slice boundaries."""
        k0, nk = self.slab(r)
        return [k0 + b for b in _split(nk, self.C, KC)]

    def sub_slab(self, rank: int) -> tuple[int, int]:
        """Slices (k0, n) rank owns at the end: sub-slab c of slab r, ceil(nk / C) slices
        each (the last ones may be shorter or empty)."""
        r, c = self.coords(rank)
        k0, nk = self.slab(r)
        q = -(-nk // self.C)
        a = min(c * q, nk)
        return k0 + a, min(q, nk - a)


def grid_groups(grid: GridPlan):
    """Row and column process groups of the grid (every rank must call this, in order).
    Returns (rows, cols): rows[r] spans ranks rC .. rC+C-1, cols[c] ranks c, c+C, ..."""
    import torch.distributed as dist

    rows = [dist.new_group([r * grid.C + c for c in range(grid.C)]) for r in range(grid.R)]
    cols = [dist.new_group([r * grid.C + c for r in range(grid.R)]) for c in range(grid.C)]
    return rows, cols


def hybrid_reconstruct(g, raw_local, vol_sub, grid: GridPlan, rank: int, row_group, col_group,
                       filter_fn: Optional[Callable] = None, bp_fn: Optional[Callable] = None,
                       timings: Optional[dict] = None, exchange: str = "auto",
                       peer: Optional[PeerExchange] = None, slabs=None, mode: int = 0,
                       streams=None):
    """R x C FDK on one rank.  raw_local: the rank's blocks of its column
    (grid.column_plan(c).local_views(r)) in order; vol_sub: [n][Ny][Nx] for
    grid.sub_slab(rank), overwritten.  Equal to one GPU up to fp32 summation order (the C
    column partial sums are added by the reduce-scatter).

    slabs (a ReduceSlabs over row r's C ranks, k_bounds = grid.sub_bounds(r)): the row sum is
    fused into the back-projection instead -- every 128-view partial sum is added straight into
    the owner of its sub-slab (ifdk_backproject_reduce), no partial slab and no reduce-scatter.
    The owner slabs must be zeroed, and every rank's adds finished, around the call (the
    caller orders them); vol_sub is unused and the own sub-slab (slabs.slab()) holds the result."""
    import torch
    import torch.distributed as dist

    r, c = grid.coords(rank)
    plan = grid.column_plan(c)
    if slabs is not None:
        from .ifdk import ifdk_backproject_reduce

        kb = grid.sub_bounds(r)
        if list(slabs.k_bounds) != kb:
            raise ValueError("slabs must be the row's chunk-aligned sub-slabs (grid.sub_bounds)")

        bases, k0s = slabs.dests()

        def fused_bp(Qb, s0, vol, k0, v0, acc):
            ifdk_backproject_reduce(g, Qb, s0, bases, k0s, k0=kb[0], nk=kb[-1] - kb[0], v0=v0,
                                    mode=mode)

        _pipeline(g, plan, r, None, col_group, filter_fn, fused_bp, timings,
                  raw_local=raw_local, exchange=exchange, peer=peer, streams=streams)
        return slabs.slab()
    k0, nk = grid.slab(r)
    q = -(-nk // grid.C)
    partial = raw_local.new_empty((q * grid.C, g.Ny, g.Nx))
    partial[nk:].zero_()  # padding rows of the reduce-scatter
    _pipeline(g, plan, r, partial[:nk], col_group, filter_fn, bp_fn, timings,
              raw_local=raw_local, exchange=exchange, peer=peer)
    sk0, sn = grid.sub_slab(rank)
    if grid.C > 1:
        out = raw_local.new_empty((q, g.Ny, g.Nx))
        dist.reduce_scatter_tensor(out, partial, op=dist.ReduceOp.SUM, group=row_group)
        vol_sub.copy_(out[:sn])
    else:
        vol_sub.copy_(partial[:sn])
    return vol_sub


def projection_split_reconstruct(g, raw_local, blocks, vol_slab, world: int, group=None,
                                 filter_fn: Optional[Callable] = None,
                                 bp_fn: Optional[Callable] = None,
                                 timings: Optional[dict] = None):
    """Projection split: rank r filters and back-projects its own views (``blocks``: the
    (first global view, count) runs stored in raw_local, in order) into a full partial volume,
    then a reduce-scatter (sum) leaves it the contiguous k-slab r (Nz divisible by world).
    vol_slab: [Nz/world][Ny][Nx].  Equal to one GPU up to fp32 summation order."""
    import torch
    import torch.distributed as dist

    filter_fn, bp_fn = _default_fns(g, filter_fn, bp_fn)
    if g.Nz % world:
        raise ValueError("projection split needs Nz divisible by the world size")
    cuda = vol_slab.is_cuda
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)] if (cuda and timings is not None) else None
    if ev:
        ev[0].record()
    Q = torch.empty_like(raw_local)
    full = raw_local.new_empty((g.Nz, g.Ny, g.Nx))
    if raw_local.shape[0] > 0:
        filter_fn(raw_local, Q)
    off, first = 0, True
    for s0, n in blocks:
        if n > 0:
            bp_fn(Q[off:off + n], s0, full, 0, 0, not first)
            first = False
        off += n
    if first:
        full.zero_()
    del Q
    if ev:
        ev[1].record()
    if world > 1:
        dist.reduce_scatter_tensor(vol_slab, full, op=dist.ReduceOp.SUM, group=group)
    else:
        vol_slab.copy_(full)
    if ev:
        ev[2].record()
        ev[2].synchronize()
        timings.update({"filter_bp_ms": ev[0].elapsed_time(ev[1]),
                        "reduce_scatter_ms": ev[1].elapsed_time(ev[2]),
                        "wall_ms": ev[0].elapsed_time(ev[2])})
    return vol_slab
