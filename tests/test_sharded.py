"""Multi-GPU path: Morton-range shards and their exchanges.

CPU: shard arithmetic, the halo plans, and ShardComm (all-gather, halo
exchange, phi row all-gather) over real world-size-2 and 4 gloo groups (the
same torch.distributed calls NCCL runs on the GPU box).
GPU: the full sharded matvec (a) as 2 and 4 gloo processes sharing the one
GPU (every exchange is host-staged, so no kernel ever waits on another
rank's), and (b) with 2, 3, 4 and 8 ranks emulated as host threads on one
device, both against the unsharded result.
"""

import os
import socket
import threading

import numpy as np
import pytest
import torch

from conftest import rel_l2, unit_cloud
from paper_1903_02153_b200.parallel import MortonShards, ShardComm, shard_range


def test_shard_ranges_partition_and_nest():
    for world in (1, 2, 4, 8):
        for lev in (2, 3, 5):
            cover = []
            for r in range(world):
                lo, hi = MortonShards(world, r).cells(lev)
                cover.append((lo, hi))
                plo, phi = MortonShards(world, r).cells(lev - 1) if lev > 2 else (lo // 8, hi // 8)
                assert (lo, hi) == (8 * plo, 8 * phi)  # children of the parent range
            assert cover[0][0] == 0 and cover[-1][1] == 8 ** lev
            assert all(a[1] == b[0] for a, b in zip(cover, cover[1:]))
    with pytest.raises(ValueError):
        MortonShards(3, 0)
    with pytest.raises(ValueError):
        shard_range(64, 5, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, results):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = ShardComm(dist)
    lev, row = 2, 3
    full = torch.zeros(8 ** lev * row, dtype=torch.float64)
    lo, hi = shard_range(8 ** lev, world, rank)
    full[lo * row:hi * row] = torch.arange(lo * row, hi * row, dtype=torch.float64)
    comm.allgather_cells(full, row, lev)
    phi = torch.zeros(10, dtype=torch.float64)
    phi[rank::world] = rank + 1.0
    comm.allreduce_sum(phi)
    results[rank] = (full.numpy().copy(), phi.numpy().copy())
    dist.destroy_process_group()


def test_balanced_bounds_minimise_the_largest_share():
    from paper_1903_02153_b200.parallel import balanced_bounds
    w = np.ones(64)
    assert balanced_bounds(w, 4) == (0, 16, 32, 48, 64)
    w = np.zeros(64)
    w[5] = 100.0          # one heavy cell, a light remainder
    w[40:] = 1.0
    b = balanced_bounds(w, 3)
    loads = [w[b[i]:b[i + 1]].sum() for i in range(3)]
    assert max(loads) == 100.0 and b[0] == 0 and b[-1] == 64
    assert all(b[i] < b[i + 1] for i in range(3))
    s = MortonShards(3, 1, balance="work")
    s.set_work(w)
    assert s.cells(2) == (b[1], b[2]) and s.cells(4) == (b[1] * 64, b[2] * 64)
    assert not s.equal


def _gloo_balanced_worker(rank, world, port, results):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = ShardComm(dist)
    shards = MortonShards(world, rank, balance="work")
    w = np.ones(64)
    w[:10] = 20.0
    shards.set_work(w)
    lev, row = 3, 2
    full = torch.zeros(8 ** lev * row, dtype=torch.float64)
    lo, hi = shards.cells(lev)
    full[lo * row:hi * row] = torch.arange(lo * row, hi * row, dtype=torch.float64)
    comm.allgather_cells(full, row, lev, shards)
    results[rank] = (full.numpy().copy(), shards.bounds)
    dist.destroy_process_group()


def test_unequal_shards_allgather_over_gloo_world2():
    import torch.multiprocessing as mp
    port = _free_port()
    results = mp.Manager().dict()
    mp.spawn(_gloo_balanced_worker, args=(2, port, results), nprocs=2, join=True)
    assert results[0][1] == results[1][1] and results[0][1][1] != 32
    for r in range(2):
        assert np.array_equal(results[r][0], np.arange(8 ** 3 * 2, dtype=np.float64))


def test_shard_comm_over_gloo_world2():
    import torch.multiprocessing as mp
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_gloo_worker, args=(world, port, results), nprocs=world, join=True)
    for r in range(world):
        full, phi = results[r]
        assert np.array_equal(full, np.arange(64 * 3, dtype=np.float64))
        assert np.array_equal(phi, np.array([1.0, 2.0] * 5))



# ---------------------------------------------------------------------------
# halo plans (CPU)

@pytest.mark.parametrize("world,level", [(2, 5), (4, 5), (8, 6), (8, 5)])
def test_halo_plan_covers_every_m2l_source(world, level):
    """Own cells + received halo = every source the shard's M2L reads (the
    target cells' far offsets, |t|_inf <= 3); each received cell comes from
    its owner, and what a rank sends is exactly what its peer receives."""
    from paper_1903_02153_b200.parallel import halo_plan
    from paper_1903_02153_b200.tables import OFFSETS
    shards = MortonShards(world, 0)
    n = 1 << level
    plans = [halo_plan(shards.bounds, level, r, world) for r in range(world)]
    rng = np.random.default_rng(level)

    def morton(x, y, z):
        out = 0
        for b in range(level):
            out |= (((x >> b) & 1) << (3 * b + 2)) | (((y >> b) & 1) << (3 * b + 1)) | (((z >> b) & 1) << (3 * b))
        return out
    for r in range(world):
        lo, hi = MortonShards(world, r).cells(level)
        have = set(range(lo, hi)) | set(int(c) for cs in plans[r].recv.values() for c in cs)
        for q, cells in plans[r].recv.items():
            qlo, qhi = MortonShards(world, q).cells(level)
            assert np.all((cells >= qlo) & (cells < qhi))
            assert np.array_equal(plans[q].send[r], cells)
        # sample target cells of this shard; every far source must be present
        for _ in range(60):
            x, y, z = (int(v) for v in rng.integers(0, n, 3))
            c = morton(x, y, z)
            if not lo <= c < hi:
                continue
            for t in OFFSETS:
                sx, sy, sz = x + int(t[0]), y + int(t[1]), z + int(t[2])
                if 0 <= sx < n and 0 <= sy < n and 0 <= sz < n:
                    assert morton(sx, sy, sz) in have
    if world == 8 and level == 6:  # a thin shell: most of the level is not sent
        assert plans[0].halo_cells < 0.5 * plans[0].own_cells


def _gloo_halo_worker(rank, world, port, results):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = ShardComm(dist)
    shards = MortonShards(world, rank)
    lev, row = 5, 2
    full = torch.zeros(8 ** lev * row, dtype=torch.float64)
    lo, hi = shards.cells(lev)
    full[lo * row:hi * row] = torch.arange(lo * row, hi * row, dtype=torch.float64) + 1
    comm.halo_exchange(full, row, lev, shards)
    counts = [r + 2 for r in range(world)]
    mine = torch.full((counts[rank], 3), float(rank))
    rows = comm.allgather_rows(mine, counts)
    results[rank] = (full.numpy().copy(), rows.numpy().copy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_halo_exchange_and_row_gather_over_gloo(world):
    import torch.multiprocessing as mp
    from paper_1903_02153_b200.parallel import halo_plan
    port = _free_port()
    results = mp.Manager().dict()
    mp.spawn(_gloo_halo_worker, args=(world, port, results), nprocs=world, join=True)
    lev, row = 5, 2
    ref = np.arange(8 ** lev * row, dtype=np.float64) + 1
    for r in range(world):
        full, rows = results[r]
        shards = MortonShards(world, r)
        lo, hi = shards.cells(lev)
        plan = halo_plan(shards.bounds, lev, r, world)
        have = np.zeros(8 ** lev, bool)
        have[lo:hi] = True
        for cells in plan.recv.values():
            have[cells] = True
        f = full.reshape(-1, row)
        assert np.array_equal(f[have], ref.reshape(-1, row)[have])
        assert not f[~have].any()  # nothing outside own + halo arrives
        want = np.concatenate([np.full((q + 2, 3), float(q)) for q in range(world)])
        assert np.array_equal(rows, want)


# ---------------------------------------------------------------------------
# the full sharded matvec on the GPU

class ThreadComm:
    """ShardComm stand-in for ranks running as threads on one GPU: the same
    exchanges (level all-gather, halo exchange by the same plans, phi row
    all-gather) through a host-synchronised shared board."""

    HALO_MIN_LEVEL = ShardComm.HALO_MIN_LEVEL

    def __init__(self, world, rank, board, barrier):
        self.world, self.rank, self.board, self.barrier = world, rank, board, barrier
        self.halo_calls = 0

    def _publish(self, t):
        torch.cuda.current_stream().synchronize()
        self.board[self.rank] = t
        self.barrier.wait()

    def _done(self):
        torch.cuda.current_stream().synchronize()
        self.barrier.wait()

    def allgather_cells(self, full, row_elems, level, shards=None):
        self._publish(full)
        for r in range(self.world):
            if r != self.rank:
                lo, hi = (shards.cells_of(r, level) if shards is not None
                          else shard_range(8 ** level, self.world, r))
                full[lo * row_elems:hi * row_elems].copy_(
                    self.board[r][lo * row_elems:hi * row_elems])
        self._done()
        return full

    def exchange_level(self, full, row_elems, level, shards):
        from paper_1903_02153_b200.parallel import halo_plan
        if level >= self.HALO_MIN_LEVEL:
            plan = halo_plan(shards.bounds, level, self.rank, self.world)
            if plan.halo_cells * 2 < (8 ** level - plan.own_cells):
                self.halo_calls += 1
                self._publish(full)
                rows = full.view(-1, row_elems)
                for r, cells in plan.recv.items():
                    idx = torch.from_numpy(cells).to(full.device)
                    rows.index_copy_(0, idx, self.board[r].view(-1, row_elems).index_select(0, idx))
                self._done()
                return full
        return self.allgather_cells(full, row_elems, level, shards)

    def allreduce_max(self, t):
        self._publish(t.clone())
        m = torch.stack([self.board[r] for r in range(self.world)]).amax(dim=0)
        self._done()
        t.copy_(m)
        return t

    def allgather_rows(self, mine, counts):
        self._publish(mine.clone())
        out = torch.cat([self.board[r] for r in range(self.world)])
        self._done()
        return out


def _run_threads(world, make_eval, pts, w, balance="cells"):
    board, barrier = {}, threading.Barrier(world)
    out, errs, comms = {}, [], {}

    def rank_main(r):
        try:
            ev = make_eval()
            comms[r] = ThreadComm(world, r, board, barrier)
            with torch.cuda.stream(torch.cuda.Stream()):
                out[r] = ev.evaluate(pts, weights=w,
                                     _shard=(MortonShards(world, r, balance=balance), comms[r]))
        except Exception as e:  # pragma: no cover
            errs.append(e)
            barrier.abort()

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    return out, comms


@pytest.mark.gpu
@pytest.mark.parametrize("world,scheme,far_mode,balance", [(2, "chebyshev", "dense", "cells"),
                                                           (4, "chebyshev", "dense", "cells"),
                                                           (2, "uniform", "dense", "cells"),
                                                           (4, "chebyshev", "active", "cells"),
                                                           (3, "chebyshev", "active", "work"),
                                                           (2, "uniform", "dense", "work")])
def test_sharded_matvec_matches_unsharded(world, scheme, far_mode, balance, cache_dir):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1903_02153_b200 as bf
    pts, w = unit_cloud(30000, seed=51, ncols=2)
    if far_mode == "active" or balance == "work":  # two clusters: most cells empty
        pts[:15000] = np.clip(0.3 + 0.03 * np.random.default_rng(5).standard_normal((15000, 3)), 0, 1)
        pts[15000:] = np.clip(0.8 + 0.02 * np.random.default_rng(6).standard_normal((15000, 3)), 0, 1)
    plan = bf.FmmPlan(levels=4, order=4, scheme=scheme, eps=1e-6,
                      domain_center=(0.5, 0.5, 0.5), domain_length=1.0)
    ref_ev = bf.FmmEvaluator(bf.EXPONENTIAL, plan, cache_dir=cache_dir)
    ref_ev.far_mode = "dense"
    ref = ref_ev.evaluate(pts, weights=w)

    def make():
        ev = bf.FmmEvaluator(bf.EXPONENTIAL, plan, cache_dir=cache_dir)
        ev.far_mode = far_mode
        return ev
    out, _ = _run_threads(world, make, pts, w, balance)
    for r in range(world):
        assert rel_l2(out[r], ref) < 1e-13


@pytest.mark.gpu
def test_eight_rank_c5_scaled_matches_unsharded(cache_dir):
    """C5/64 (N = 1M, L = 6, Laplace, p = 5) as 8 thread-emulated ranks: each
    owns one octant box, the fine levels exchange only their halo and run the
    plane-buffered int8 M2L on the box."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1903_02153_b200 as bf
    from paper_1903_02153_b200 import workloads
    wl = workloads.make("C5", 2)
    plan = bf.FmmPlan(levels=wl["levels"], order=wl["order"], eps=wl["eps"],
                      domain_center=wl["center"], domain_length=wl["length"])
    ref = bf.FmmEvaluator(bf.LAPLACIAN, plan, cache_dir=cache_dir).evaluate(
        wl["points"], weights=wl["weights"])
    out, comms = _run_threads(8, lambda: bf.FmmEvaluator(bf.LAPLACIAN, plan, cache_dir=cache_dir),
                              wl["points"], wl["weights"])
    for r in range(8):
        assert rel_l2(out[r], ref) < 1e-13
    assert all(c.halo_calls >= 1 for c in comms.values())  # level 6 went halo-only


def _gloo_matvec_worker(rank, world, port, scheme, cache_dir, results):
    import torch.distributed as dist

    import paper_1903_02153_b200 as bf
    from paper_1903_02153_b200.parallel import ShardedEvaluator
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pts, w = unit_cloud(40000, seed=61, ncols=1)
    plan = bf.FmmPlan(levels=5, order=4, scheme=scheme, eps=1e-6,
                      domain_center=(0.5, 0.5, 0.5), domain_length=1.0)
    ev = bf.FmmEvaluator(bf.LAPLACIAN if scheme == "chebyshev" else bf.EXPONENTIAL, plan,
                         cache_dir=cache_dir)
    runner = ShardedEvaluator(ev, dist, balance="cells")
    results[rank] = runner.evaluate(pts, weights=w[:, 0])
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,scheme", [(2, "chebyshev"), (4, "chebyshev"), (2, "uniform")])
def test_gloo_processes_sharded_matvec_matches_unsharded(world, scheme, cache_dir):
    """World-2/4 process groups (gloo, host-staged exchanges) sharing the
    one GPU run the full sharded matvec through ShardedEvaluator -- the same
    code path as the NCCL ranks of bench.py --gpus N."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    import paper_1903_02153_b200 as bf
    pts, w = unit_cloud(40000, seed=61, ncols=1)
    plan = bf.FmmPlan(levels=5, order=4, scheme=scheme, eps=1e-6,
                      domain_center=(0.5, 0.5, 0.5), domain_length=1.0)
    k = bf.LAPLACIAN if scheme == "chebyshev" else bf.EXPONENTIAL
    ref = bf.FmmEvaluator(k, plan, cache_dir=cache_dir).evaluate(pts, weights=w[:, 0])
    port = _free_port()
    results = mp.Manager().dict()
    mp.spawn(_gloo_matvec_worker, args=(world, port, scheme, cache_dir, results), nprocs=world,
             join=True)
    for r in range(world):
        assert rel_l2(results[r], ref) < 1e-13
