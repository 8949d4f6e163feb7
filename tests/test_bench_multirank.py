"""bench.py's N > 1 path (one process per GPU, z-slab sharding, per-rank int64 record gather, max-over-ranks
timing), run with 2 ranks sharing the visible GPU (SAND_BENCH_SHARE_GPU=1: gloo instead of NCCL).  The
ranks' kernels never wait on each other, so sharing one GPU is safe."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*extra, share=True, timeout=1200):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "2", "--warmup", "3", "--no-cpu", "--no-e2e",
           "--no-full-depth", *extra]
    env = dict(os.environ, SAND_BENCH_SHARE_GPU="1") if share else dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, "exactly one JSON line (rank 0)"
    return lines[0], r.stderr


def test_gpus2_self_launch_c4_strong():
    """`bench.py --gpus 2` with no torchrun environment launches 2 ranks itself; the default N > 1 workload is
    BASELINE.json configs[4]: the fixed 1024^3 grid (level-8 octree) strong-scaled over work-balanced z-slabs."""
    d, err = _bench("--gpus", "2")
    assert "torch.distributed.run" in err and "nranks=2" in err
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["global_points"] == 1024 ** 3
    assert sum(d["per_depth"]) == 1024 ** 3                   # every point binned once
    (a0, b0), (a1, b1) = d["shards"]
    assert a0 == 0 and b0 == a1 and b1 == 1024
    assert d["comm"]["nranks"] == 2
    assert d["value"] > 0 and d["roofline"]["frac"] > 0


def test_checksums_identical_for_one_and_two_ranks():
    """SURVEY 8(e) pin through the bench: C1 strong-scaled over 2 ranks gives the same int64 fixed-point SDF
    checksum, depth hash and per-depth counts as 1 rank (every point's math is independent of its shard)."""
    d2, _ = _bench("--gpus", "2", "--config", "C1")
    d1, _ = _bench("--gpus", "1", "--config", "C1", share=False)
    assert d2["n_gpus"] == 2 and d1["n_gpus"] == 1
    assert d2["checksums"]["sdf_fixed_point_2^24"] == d1["checksums"]["sdf_fixed_point_2^24"]
    assert d2["checksums"]["depth_hash"] == d1["checksums"]["depth_hash"]
    assert d2["per_depth"] == d1["per_depth"]


def test_weak_scaling_option():
    d, _ = _bench("--gpus", "2", "--config", "C1", "--scaling", "weak")
    assert d["scaling"] == "weak" and d["config"]["global_points"] == 2 * 256 ** 3
