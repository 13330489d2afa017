"""Multi-GPU path: Morton-range shards and their two exchanges.

CPU: shard arithmetic, and ShardComm over a real world-size-2 gloo group
(the same torch.distributed calls NCCL runs on the GPU box).
GPU: the sharded matvec with 2 and 4 ranks emulated as host threads on one
device (each rank on its own stream; the exchanges synchronise on the host,
no kernel ever waits on another rank), against the unsharded result.
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


class ThreadComm:
    """ShardComm stand-in for ranks running as threads on one GPU."""

    def __init__(self, world, rank, board, barrier):
        self.world, self.rank, self.board, self.barrier = world, rank, board, barrier

    def allgather_cells(self, full, row_elems, level, shards=None):
        torch.cuda.current_stream().synchronize()
        self.board[self.rank] = full
        self.barrier.wait()
        for r in range(self.world):
            if r != self.rank:
                lo, hi = (shards.cells_of(r, level) if shards is not None
                          else shard_range(8 ** level, self.world, r))
                full[lo * row_elems:hi * row_elems].copy_(
                    self.board[r][lo * row_elems:hi * row_elems])
        torch.cuda.current_stream().synchronize()
        self.barrier.wait()
        return full

    def allreduce_sum(self, t):
        torch.cuda.current_stream().synchronize()
        self.board[self.rank] = t.clone()
        self.barrier.wait()
        total = sum(self.board[r] for r in range(self.world))
        self.barrier.wait()
        t.copy_(total)
        return t


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
    board, barrier = {}, threading.Barrier(world)
    out, errs = {}, []

    def rank_main(r):
        try:
            ev = bf.FmmEvaluator(bf.EXPONENTIAL, plan, cache_dir=cache_dir)
            ev.far_mode = far_mode
            with torch.cuda.stream(torch.cuda.Stream()):
                out[r] = ev.evaluate(pts, weights=w,
                                     _shard=(MortonShards(world, r, balance=balance),
                                             ThreadComm(world, r, board, barrier)))
        except Exception as e:  # pragma: no cover
            errs.append(e)
            barrier.abort()

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for r in range(world):
        assert rel_l2(out[r], ref) < 1e-13
