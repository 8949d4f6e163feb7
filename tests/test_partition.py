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
    from oracle import fp32 as ofp
    c = g.make_config("C0")
    p = c.params()
    k0, k1, Rz = partition.shard_planes(c.depthmap, R, world, rank, weak=False)
    pts = g.grid_points_slab(R, k0, k1, Rz)
    sdf, d = ofp.query_fp32(p, c.depthmap, pts)
    per_depth = np.bincount(d, minlength=c.spec.L + 1)
    gidx = np.arange(pts.shape[0], dtype=np.int64) + k0 * R * R
    sdf_fx = int(np.round(sdf.astype(np.float64) * (1 << 24)).astype(np.int64).sum())
    dhash = int((d.astype(np.int64) * (gidx % 8191 + 1)).sum())
    rec = partition.make_record(pts.shape[0], per_depth, 1.0 + rank, sdf_fx, dhash, k0, k1, 1)
    t = torch.from_numpy(rec)
    allr = torch.empty(world * t.numel(), dtype=t.dtype)
    dist.all_gather_into_tensor(allr, t)
    if rank == 0:
        out.put(partition.summarize(allr.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def _run_world(world, R):
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
    return summ


def test_gloo_world2_shards_tile_grid_and_checksums_match_one_rank():
    """Strong sharding of C0's 64^3 grid over 2 gloo ranks: the shards tile the grid once, the gathered
    per-depth counts equal the single-process lookup's, and the int64 fixed-point SDF checksum and the
    global-index depth hash summed over ranks are bit-identical to the 1-rank run (SURVEY 8(e) pin)."""
    R = 64
    summ2 = _run_world(2, R)
    summ1 = _run_world(1, R)
    ranges = summ2["ranges"]
    assert ranges[0][0] == 0 and ranges[-1][1] == R and ranges[0][1] == ranges[1][0]
    c = g.make_config("C0")
    d, _, _ = oracle.lookup(c.depthmap, c.points_fn())
    assert summ2["n_total"] == R ** 3
    np.testing.assert_array_equal(summ2["per_depth"][:c.spec.L + 1], np.bincount(d, minlength=c.spec.L + 1))
    assert summ2["ms_max"] == 2.0 and summ2["ms_min"] == 1.0
    assert summ2["sdf_fx"] == summ1["sdf_fx"] and summ2["depth_hash"] == summ1["depth_hash"]
    assert summ2["per_depth"] == summ1["per_depth"]


def test_record_is_int64_and_exact():
    rec = partition.make_record(10, [1, 2, 3], 1.5, -(1 << 60), 123456789012345, 3, 7, 2, 4.25)
    assert rec.dtype == np.int64
    s = partition.summarize(np.concatenate([rec, rec]))
    assert s["sdf_fx"] == -(1 << 61) and s["depth_hash"] == 2 * 123456789012345
    assert s["ms_max"] == 1.5 and s["ms_full_max"] == 4.25 and s["n_total"] == 20


@pytest.mark.parametrize("world", [2, 4, 8])
def test_c4_strong_partition_balanced(world):
    """BASELINE.json configs[4]: the fixed 1024^3 grid cut into `world` z-slabs by estimated work: every plane
    once, and the estimated max/mean work <= 1.01 (equal-thickness slabs: 1.16 at 8 ranks)."""
    c = g.make_config("C4")
    R = c.grid_R
    w = partition.plane_work(c.depthmap, R, R)
    sl = [partition.shard_planes(c.depthmap, R, world, r, weak=False) for r in range(world)]
    assert all(Rz == R for _, _, Rz in sl)
    assert sl[0][0] == 0 and sl[-1][1] == R and all(sl[r][1] == sl[r + 1][0] for r in range(world - 1))
    per = np.array([w[k0:k1].sum() for k0, k1, _ in sl])
    assert per.max() / per.mean() <= 1.01


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
