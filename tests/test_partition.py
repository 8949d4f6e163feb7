"""Multi-GPU host logic on CPU: work-balanced z-slab sharding and the per-rank
record all-gather, exercised with torch.distributed `gloo` at world_size 2 (the GPU run uses the
same code with backend `nccl`).  Points are independent (Sec. 3.4), so the
shards must tile the grid exactly once and the gathered per-depth counts must equal the
single-process ones."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import sandgen as g
from paper_2604_25936_b200 import partition


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_balanced_cuts_cover_and_balance():
    rng = np.random.default_rng(0)
    w = rng.gamma(0.5, 1.0, 1000)
    for parts in (1, 2, 3, 8):
        c = partition.balanced_cuts(w, parts)
        assert c[0] == 0 and c[-1] == w.size and np.all(np.diff(c) >= 1)
        sums = np.add.reduceat(w, c[:-1])
        # each part is within one plane's work of the ideal share
        assert np.all(np.abs(sums - w.sum() / parts) <= w.max() + 1e-9)
    with pytest.raises(ValueError):
        partition.balanced_cuts(np.ones(3), 4)


def test_plane_work_matches_exact_per_plane_depth_sums():
    """The work model's per-plane depth sum equals the oracle lookup's exact per-plane sum."""
    c = g.make_config("C0")
    R = c.grid_R
    pts = c.points_fn()
    d, _, _ = oracle.lookup(c.depthmap, pts)
    exact = (d.astype(np.float64) + 0.5).reshape(R, R * R).sum(1)
    est = partition.plane_work(c.depthmap, R, R, eps=0.5)
    np.testing.assert_allclose(est, exact, rtol=1e-12)


def _worker(rank, world, port, R, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = g.make_config("C0")
    k0, k1, Rz = partition.shard_planes(c.depthmap, R, world, rank, weak=False)
    pts = g.grid_points_slab(R, k0, k1, Rz)
    d, _, _ = oracle.lookup(c.depthmap, pts)
    per_depth = np.bincount(d, minlength=c.spec.L + 1)
    rec = partition.make_record(pts.shape[0], per_depth, 1.0 + rank, float(pts.astype(np.float64).sum()),
                                float(d.sum()), k0, k1, 1)
    t = torch.from_numpy(rec)
    allr = torch.empty(world * t.numel(), dtype=t.dtype)
    dist.all_gather_into_tensor(allr, t)
    if rank == 0:
        out.put(partition.summarize(allr.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_shards_tile_grid_and_gather_matches_single_process():
    R, world = 64, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, R, q)) for r in range(world)]
    for p in procs:
        p.start()
    summ = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    ranges = summ["ranges"]
    assert ranges[0][0] == 0 and ranges[-1][1] == R and ranges[0][1] == ranges[1][0]
    c = g.make_config("C0")
    pts = c.points_fn()
    d, _, _ = oracle.lookup(c.depthmap, pts)
    assert summ["n_total"] == R ** 3
    np.testing.assert_array_equal(summ["per_depth"][:c.spec.L + 1], np.bincount(d, minlength=c.spec.L + 1))
    assert summ["ms_max"] == 2.0 and summ["ms_min"] == 1.0
    np.testing.assert_allclose(summ["checksum"], pts.astype(np.float64).sum(), rtol=1e-12)


def test_weak_scaling_shards_hold_about_R3_points_each():
    c = g.make_config("C2")
    R, world = 512, 8
    sizes = []
    for r in range(world):
        k0, k1, Rz = partition.shard_planes(c.depthmap, R, world, r, weak=True)
        assert Rz == R * world
        sizes.append(k1 - k0)
    assert sum(sizes) == R * world
    # work balance: estimated per-rank work within 2% of the mean
    w = partition.plane_work(c.depthmap, R, R * world)
    cuts = np.concatenate([[0], np.cumsum(sizes)])
    per = np.array([w[cuts[i]:cuts[i + 1]].sum() for i in range(world)])
    assert per.max() / per.mean() < 1.02
