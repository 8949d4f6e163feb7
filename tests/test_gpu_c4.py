"""BASELINE.json configs[4] ("C4": 8x256 BF16 net, C2's octree extended to level 8, the 1024^3 grid) on the
GPU: every point's exit depth against the FP32 C oracle (streamed in z-slabs), a stratified SDF sample, and
shard invariance across the work-balanced cut planes the 8-rank bench uses (SURVEY 8(e) pin)."""
import numpy as np
import pytest

import sandgen as g
from _engine import TOL_BF16, assert_parity, make_ctx, oracle_query, stratified_sample
from oracle import fp32 as ofp
from paper_2604_25936_b200 import partition

pytestmark = pytest.mark.gpu
BF16 = 2


def _query(ctx, pts_np):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(pts_np)).cuda()
    sdf, dep = ctx.query_tensor(t)
    torch.cuda.synchronize()
    return sdf.cpu().numpy(), dep.cpu().numpy()


@pytest.fixture(scope="module")
def c4():
    c = g.make_config("C4")
    p = c.params()
    ctx = make_ctx(c.spec, BF16)
    ctx.sand_load_weights(g.pack_blob(p))
    ctx.sand_load_depthmap(c.depthmap)
    ctx.sand_reserve(64 * 1024 * 1024)
    yield c, p, ctx
    ctx.close()


def test_c4_all_exit_depths_and_sdf_sample(c4):
    c, p, ctx = c4
    R = c.grid_R
    step = 64
    sdf_idx = []
    for k0 in range(0, R, step):
        pts = g.grid_points_slab(R, k0, k0 + step)
        sdf, dep = _query(ctx, pts)
        np.testing.assert_array_equal(dep, ofp.lookup_fp32(c.depthmap, pts))
        if k0 % 256 == 0:   # SDF: a stratified sample (all depths) of every fourth slab
            idx = stratified_sample(dep, 2048, 8192, seed=k0)
            sdf_or, dep_or = oracle_query(p, c.depthmap, pts[idx])
            assert_parity(sdf, dep, sdf_or, dep_or, TOL_BF16, idx=idx)
            sdf_idx.append(idx.size)
    assert sum(sdf_idx) > 0


def test_c4_shard_invariance_at_8_rank_cuts(c4):
    """Planes around every cut of the 8-rank strong partition: querying the two sides separately (as two
    ranks do) reproduces the joint query bit for bit."""
    c, p, ctx = c4
    R = c.grid_R
    cuts = [partition.shard_planes(c.depthmap, R, 8, r, weak=False)[0] for r in range(1, 8)]
    for k in cuts:
        pts = g.grid_points_slab(R, k - 3, k + 3)
        s_all, d_all = _query(ctx, pts)
        half = 3 * R * R
        s_lo, d_lo = _query(ctx, pts[:half])
        s_hi, d_hi = _query(ctx, pts[half:])
        np.testing.assert_array_equal(np.concatenate([d_lo, d_hi]), d_all)
        np.testing.assert_array_equal(np.concatenate([s_lo, s_hi]), s_all)
