"""Multi-rank host logic of the k-slab and projection-split drivers, world size 2 to 4
over gloo on CPU (the fused exchange's round protocol through a shared-memory fake of
dist.PeerExchange).  The compute is injected (fp64 oracle filter / back-projection), so
these tests check the plan, the row-band all-to-all and the reduce-scatter bookkeeping;
the oracle raises if any rank is missing a detector row its slab taps."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
import synth
from paper_1909_02724_b200 import Geometry
from paper_1909_02724_b200.dist import (GridPlan, SlabPlan, grid_groups, hybrid_reconstruct,
                                        kslab_reconstruct, kslab_reconstruct_host, plan_exchange,
                                        projection_split_fused, projection_split_reconstruct)

SPEC = synth.ConfigSpec("dist 36x40x36->24x20x40", 36, 40, 36, 24, 20, 40)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_fns(og):
    def filter_fn(raw, out):
        out.copy_(torch.from_numpy(oracle.filter_fft(og, raw.numpy()).astype(np.float32)))

    def bp_fn(Q, s0, vol, k0, v0, acc):
        part = oracle.backproject_volume(og, Q.numpy().astype(np.float64), s0=s0, v0=v0, k0=k0,
                                         nk=vol.shape[0])
        t = torch.from_numpy(part.astype(np.float32))
        if acc:
            vol.add_(t)
        else:
            vol.copy_(t)

    return filter_fn, bp_fn


def _reference():
    og = oracle.OracleGeometry(**SPEC.geometry_args())
    E = synth.project(SPEC.Nu, SPEC.Nv, SPEC.Du, SPEC.Dv, SPEC.D, SPEC.d, SPEC.theta,
                      synth.default_ellipsoids(SPEC), 0, SPEC.Np)
    Q32 = oracle.filter_fft(og, E).astype(np.float32)
    return E, oracle.backproject_volume(og, Q32.astype(np.float64))


class HostPeerExchange:
    """Host fake of dist.PeerExchange for the gloo tests: the same round protocol (wait_free,
    scatter, wait_landed, release) and buffer layout, with POSIX shared memory standing in for
    the NVLink-mapped receive buffers and host spin-waits for ifdk_wait.  Each signal word has
    a single writer (rank r writes landed[r] / freed[r] in every buffer), as on the GPU."""

    kind = "host-fake"

    def __init__(self, tag, rank, world, recv_max):
        import time
        from multiprocessing import shared_memory

        import torch.distributed as dist

        self.rank, self.world, self.recv_max = rank, world, list(recv_max)
        self._time = time
        hdr = 2 * world * 8
        self.shm = [None] * world
        self.shm[rank] = shared_memory.SharedMemory(
            name=f"{tag}_{rank}", create=True, size=hdr + 8 * max(recv_max[rank], 1))
        self.shm[rank].buf[:hdr] = bytes(hdr)
        dist.barrier()
        for h in range(world):
            if h != rank:
                self.shm[h] = shared_memory.SharedMemory(name=f"{tag}_{h}")
        self.words = [np.ndarray((2, world), np.int64, buffer=m.buf) for m in self.shm]
        self.area = [np.ndarray((2 * max(recv_max[h], 1),), np.float32, buffer=m.buf, offset=hdr)
                     for h, m in enumerate(self.shm)]
        dist.barrier()

    def close(self):
        import torch.distributed as dist

        self.words = self.area = None
        dist.barrier()
        for h, m in enumerate(self.shm):
            m.close()
            if h == self.rank:
                m.unlink()

    def _wait(self, row, target):
        t0 = self._time.time()
        while (self.words[self.rank][row] < target).any():
            if self._time.time() - t0 > 120:
                raise TimeoutError(f"rank {self.rank}: signal row {row} never reached {target}")
            self._time.sleep(0.0005)

    rounds_done = 0  # as dist.PeerExchange: the words count on across pipeline calls

    def wait_free(self, t):
        target = self.rounds_done + (t - 1 if t >= 2 else 0)
        if target > 0:
            self._wait(1, target)

    def scatter(self, g, src, q, bands, filter_fn):
        if src is not None and bands:
            Q = torch.empty_like(src)
            filter_fn(src, Q)
            n = src.shape[0]
            for h, off, lo, hi in bands:
                a = q * self.recv_max[h] + off
                dst = self.area[h][a:a + n * (hi - lo + 1) * g.Nu]
                dst.reshape(n, hi - lo + 1, g.Nu)[:] = Q[:, lo:hi + 1, :].numpy()
        for h in range(self.world):  # stores first, then the single-writer landed word
            self.words[h][0, self.rank] += 1

    def wait_landed(self, t):
        self._wait(0, self.rounds_done + t + 1)

    def recv(self, q, off, rn, rows, Nu):
        a = q * self.recv_max[self.rank] + off
        return torch.from_numpy(self.area[self.rank][a:a + rn * rows * Nu].reshape(rn, rows, Nu))

    def release(self):
        for h in range(self.world):
            self.words[h][1, self.rank] += 1


class HostReduceSlabs:
    """Host fake of dist.ReduceSlabs for the gloo tests: every rank's owner slab in POSIX shared
    memory, mapped by all ranks; the adds of the fused reduce (the GPU's red.global.add) are
    serialised by a file lock."""

    def __init__(self, tag, rank, world, k_bounds, Ny, Nx):
        import fcntl
        from multiprocessing import shared_memory

        import torch.distributed as dist

        self.rank, self.world, self.k_bounds = rank, world, list(k_bounds)
        self.Ny, self.Nx, self._fcntl = Ny, Nx, fcntl
        nk = [k_bounds[h + 1] - k_bounds[h] for h in range(world)]
        self.shm = [None] * world
        self.shm[rank] = shared_memory.SharedMemory(name=f"{tag}_{rank}", create=True,
                                                    size=4 * max(nk[rank], 1) * Ny * Nx)
        dist.barrier()
        for h in range(world):
            if h != rank:
                self.shm[h] = shared_memory.SharedMemory(name=f"{tag}_{h}")
        self.arr = [np.ndarray((nk[h], Ny, Nx), np.float32, buffer=self.shm[h].buf)
                    for h in range(world)]
        self.lock = open(f"/tmp/{tag}.lock", "w")

    def slab(self, h=None):
        return torch.from_numpy(self.arr[self.rank if h is None else h])

    def add(self, vol, k0):
        """Add a partial volume of slices k0.. into the owners' slabs (under the lock)."""
        self._fcntl.flock(self.lock, self._fcntl.LOCK_EX)
        try:
            for h in range(self.world):
                a, b = self.k_bounds[h], self.k_bounds[h + 1]
                lo, hi = max(a, k0), min(b, k0 + vol.shape[0])
                if hi > lo:
                    self.arr[h][lo - a:hi - a] += vol[lo - k0:hi - k0]
        finally:
            self._fcntl.flock(self.lock, self._fcntl.LOCK_UN)

    def close(self):
        import torch.distributed as dist

        dist.barrier()
        self.arr = []
        for h, m in enumerate(self.shm):
            m.close()
            if h == self.rank:
                m.unlink()


def _worker(rank, world, port, mode, out_q):
    import torch.distributed as dist

    os.environ["OMP_NUM_THREADS"] = "1"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        og = oracle.OracleGeometry(**SPEC.geometry_args())
        g = Geometry.from_spec(SPEC)
        f, b = _oracle_fns(og)
        E, ref = _reference()
        if mode in ("kslab", "kslab_host", "kslab_fused"):
            # 8-view blocks: 5 blocks of 36 views, several pipelined rounds and a short last one
            plan = SlabPlan(world, SPEC.Nz, SPEC.Np, block=8)
            k0, nk = plan.slab(rank)
            mine = np.concatenate([E[s0:s0 + n] for s0, n in plan.local_views(rank)])
            assert mine.shape[0] == plan.n_local(rank)
            vol = torch.empty((nk, SPEC.Ny, SPEC.Nx))
            if mode == "kslab":
                kslab_reconstruct(g, torch.from_numpy(mine), vol, plan, rank, filter_fn=f, bp_fn=b)
            elif mode == "kslab_fused":
                # the fused exchange's round protocol (dist.PeerExchange) with the host fake
                from paper_1909_02724_b200.dist import exchanges

                rmax = [max(sum(e.recv_sizes) for e in exchanges(g, plan, h)) for h in range(world)]
                peer = HostPeerExchange(f"ifdk_{port}", rank, world, rmax)
                try:
                    for _ in range(2):  # the second call counts on from the first's signals
                        vol.fill_(float("nan"))
                        kslab_reconstruct(g, torch.from_numpy(mine), vol, plan, rank,
                                          filter_fn=f, bp_fn=b, peer=peer)
                    assert peer.rounds_done == 2 * plan.n_rounds
                finally:
                    peer.close()
            else:
                host = torch.full((nk, SPEC.Ny, SPEC.Nx), float("nan"))
                kslab_reconstruct_host(g, torch.from_numpy(mine), vol, host, plan, rank,
                                       filter_fn=f, bp_fn=b)
                assert torch.equal(host, vol)
        elif mode.startswith("grid"):
            R, C = int(mode[4]), int(mode[5])
            grid = GridPlan(R, C, SPEC.Nz, SPEC.Np, block=8)
            rows, cols = grid_groups(grid)
            r, c = grid.coords(rank)
            blocks = grid.column_plan(c).local_views(r)
            mine = np.concatenate([E[s0:s0 + n] for s0, n in blocks]) if blocks else \
                np.zeros((0, SPEC.Nv, SPEC.Nu), np.float32)
            k0, nk = grid.sub_slab(rank)
            vol = torch.empty((nk, SPEC.Ny, SPEC.Nx))
            hybrid_reconstruct(g, torch.from_numpy(mine), vol, grid, rank, rows[r], cols[c],
                               filter_fn=f, bp_fn=b)
        elif mode == "psplit_fused":
            # the fused projection split: each rank's partial sums added straight into the
            # owners' slabs (here a shared-memory fake of ReduceSlabs), with its zero / barrier
            # protocol; 8-view blocks dealt round-robin as on the GPU
            plan = SlabPlan(world, SPEC.Nz, SPEC.Np, block=8)
            k0, nk = plan.slab(rank)
            blocks = plan.local_views(rank)
            mine = np.concatenate([E[s0:s0 + n] for s0, n in blocks])
            slabs = HostReduceSlabs(f"ifdkr_{port}", rank, world, plan.k_bounds, SPEC.Ny, SPEC.Nx)
            try:
                def reduce_fn(Qb, s0):
                    part = oracle.backproject_volume(og, Qb.numpy().astype(np.float64), s0=s0)
                    slabs.add(part.astype(np.float32), 0)

                own = projection_split_fused(g, torch.from_numpy(mine), blocks, slabs,
                                             filter_fn=f, reduce_fn=reduce_fn)
                vol = own.clone()
            finally:
                slabs.close()
        else:
            n = SPEC.Np // world
            s0 = rank * n
            k0, nk = rank * SPEC.Nz // world, SPEC.Nz // world
            vol = torch.empty((nk, SPEC.Ny, SPEC.Nx))
            projection_split_reconstruct(g, torch.from_numpy(E[s0:s0 + n].copy()), [(s0, n)], vol,
                                         world, filter_fn=f, bp_fn=b)
        d = vol.numpy().astype(np.float64) - ref[k0:k0 + nk]
        out_q.put((rank, float(np.abs(d).max() / np.abs(ref).max()) if d.size else 0.0))
    except Exception as e:  # surface the failure in the parent
        out_q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mode", [(2, "kslab"), (3, "kslab"), (2, "kslab_host"),
                                        (2, "kslab_fused"), (3, "kslab_fused"),
                                        (4, "kslab_fused"),
                                        (2, "projsplit"), (2, "psplit_fused"),
                                        (3, "psplit_fused"), (4, "grid22"), (3, "grid13"),
                                        (3, "grid31")])
def test_multi_rank_matches_single(world, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    for r in range(world):
        assert isinstance(res[r], float), res[r]
        assert res[r] <= 1e-6, (r, res[r])


def test_slab_plan_alignment_and_exchange_bands():
    for world in (1, 2, 4, 8):
        plan = SlabPlan(world, 2048, 2048)
        kb = plan.k_bounds
        assert kb[0] == 0 and kb[-1] == 2048
        assert all(k % 64 == 0 for k in kb)
        assert all(b > a for a, b in zip(kb[:-1], kb[1:]))
        # every view is owned exactly once, blocks start on the 128-view summation batch,
        # and round t covers the consecutive views of blocks tP .. tP+P-1
        views = sorted(v for r in range(world) for s0, n in plan.local_views(r)
                       for v in range(s0, s0 + n))
        assert views == list(range(2048))
        assert all(s0 % 128 == 0 for r in range(world) for s0, _ in plan.local_views(r))
        for t in range(plan.n_rounds):
            blocks = [plan.round_block(t, r) for r in range(world)]
            assert all(b[0] == blocks[0][0] + 128 * i for i, b in enumerate(blocks))
    plan = SlabPlan(3, 40, 36, block=8)
    assert plan.k_bounds[-1] == 40 and sum(plan.slab(r)[1] for r in range(3)) == 40
    assert plan.n_rounds == 2 and plan.round_block(1, 1) == (32, 4) and plan.round_block(1, 2)[1] == 0
    g = Geometry.from_spec(SPEC)
    for t in range(plan.n_rounds):
        ex = [plan_exchange(g, plan, r, t) for r in range(3)]
        for r in range(3):
            for h in range(3):
                # what r sends to h is what h expects from r
                assert ex[r].send[h] == ex[h].recv[r]
                assert ex[r].send_sizes[h] == ex[h].recv_sizes[r]


def test_grid_plan_partitions():
    """Every (view, slice) pair is covered exactly once: columns partition the view blocks,
    rows partition the slices, and the sub-slabs of a row partition its slab."""
    for R, C in ((1, 8), (2, 4), (4, 2), (8, 1), (3, 2)):
        grid = GridPlan(R, C, 2048, 2048)
        views = sorted(v for c in range(C) for r in range(R)
                       for s0, n in grid.column_plan(c).local_views(r) for v in range(s0, s0 + n))
        assert views == list(range(2048)), (R, C)
        ks = sorted(k for rank in range(R * C) for k in range(*(lambda a, n: (a, a + n))(
            *grid.sub_slab(rank))))
        assert ks == list(range(2048)), (R, C)
        assert all(grid.slab(r)[0] % 64 == 0 for r in range(R))
        # the fused row reduce's owner sub-slabs: partition each slab, chunk-aligned here
        for r in range(R):
            kb = grid.sub_bounds(r)
            assert kb[0] == grid.slab(r)[0] and kb[-1] == sum(grid.slab(r))
            assert all(a <= b for a, b in zip(kb, kb[1:])) and all(k % 64 == 0 for k in kb)


def test_reduce_slab_destinations_skip_empty_slabs():
    """ReduceSlabs.dests (what ifdk_backproject_reduce receives): the non-empty owner slabs, in
    order, with strictly increasing first slices -- e.g. 8 ranks over 320 slices or over 100
    (ranks without slices own an empty slab)."""
    from paper_1909_02724_b200.dist import ReduceSlabs

    for world, Nz in ((8, 320), (8, 100), (3, 2048), (1, 7)):
        kb = SlabPlan(world, Nz, 64).k_bounds
        rs = ReduceSlabs(0, world, list(range(1000, 1000 + world)), kb, 4, 4)
        bases, k0s = rs.dests()
        assert k0s[0] == 0 and all(a < b for a, b in zip(k0s, k0s[1:]))
        assert len(bases) == sum(1 for h in range(world) if kb[h + 1] > kb[h])
        assert all(kb[bases[i] - 1000] == k0s[i] for i in range(len(bases)))


def test_band_exchange_volume_config4_p8():
    """At config 4 on 8 ranks the rows exchanged per rank stay far below a full all-gather
    (band <= ~0.15 Nv per view)."""
    spec = synth.config(4)
    g = Geometry.from_spec(spec)
    plan = SlabPlan(8, spec.Nz, spec.Np)
    rows = 0
    for t in range(plan.n_rounds):
        ex = plan_exchange(g, plan, 0, t)
        rows += sum(ex.views[r][1] * (hi - lo + 1) for r, (lo, hi) in enumerate(ex.recv))
    full = spec.Np * spec.Nv
    assert rows / full < 0.2, rows / full


def test_d2h_pieces_cover_the_slab_on_chunk_boundaries():
    """The end-to-end driver's D2H pieces tile the slab exactly, start on multiples of 64
    slices relative to the slab start (the BP chunk, so sub-slab launches leave the result
    unchanged) and end with pieces of at most D2H_TAIL slices."""
    from paper_1909_02724_b200.dist import D2H_SUBSLAB, D2H_TAIL, _d2h_pieces

    for k0, nk in ((0, 2048), (256, 256), (0, 100), (64, 600), (512, 513), (0, 1)):
        pieces = _d2h_pieces(k0, nk)
        a = k0
        for s, n in pieces:
            assert s == a and 0 < n <= D2H_SUBSLAB and (s - k0) % 64 == 0
            a += n
        assert a == k0 + nk
        tail = [n for s, n in pieces if s >= k0 + nk - D2H_SUBSLAB]
        assert all(n <= D2H_TAIL for n in tail)
