"""GPU parity: libsand (CUDA, via the C ABI) vs the oracle on the same seeded inputs.

Bar (BASELINE.json north_star): exit depths bit-exact on every compared point; SDF max-abs <= 5e-3
(BF16 path) / 1e-4 (FP32 path); sign agreement wherever |oracle| > 5e-3.
"""
import os

import numpy as np
import pytest

import oracle
import sandgen as g
from _engine import (TOL_BF16, TOL_FP32, assert_parity, make_ctx, oracle_query, run_engine,
                     stratified_sample)

pytestmark = pytest.mark.gpu

BF16, FP32 = 2, 0


def _random_voxel_map(level, L, seed, far=False):
    rng = np.random.default_rng(seed)
    G = 1 << level
    lo = 0 if far else 1
    dep = rng.integers(lo, L + 1, G ** 3).astype(np.uint8)
    fs = rng.normal(size=G ** 3).astype(np.float32) if far else None
    return g.VoxelMap(level, dep, fs)


def _pts(n, seed, lo=-1.0, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, (n, 3)).astype(np.float32)


@pytest.mark.parametrize("H", [64, 128, 256, 336])
@pytest.mark.parametrize("tail", [0, 1])
def test_bf16_random_depths_small(H, tail):
    """All depths 1..L mixed, several tiles per depth with ragged tails, n not a multiple of 4."""
    L = 5
    spec = g.TMlpSpec(L=L, H=H, omega0=30.0, tail=tail, seed=4)
    p = g.make_weights(spec)
    dm = _random_voxel_map(3, L, 1)
    pts = _pts(7001, 2)
    with make_ctx(spec, BF16) as ctx:
        sdf, dep = run_engine(ctx, p, dm, pts)
    sdf_or, dep_or = oracle_query(p, dm, pts)
    assert_parity(sdf, dep, sdf_or, dep_or, TOL_BF16)


@pytest.mark.parametrize("L", [1, 2, 8])
def test_bf16_wide_pair_kernel(L):
    """H = 336 (configs[3] width) on the wide CTA-pair kernel: single-layer and two-layer edge cases and
    the full L = 8 net, many 256-row tiles per depth with ragged tails."""
    spec = g.TMlpSpec(L=L, H=336, omega0=30.0, tail=0, seed=40 + L)
    p = g.make_weights(spec)
    dm = _random_voxel_map(3, L, 11)
    pts = _pts(60007, 12)
    with make_ctx(spec, BF16) as ctx:
        sdf, dep = run_engine(ctx, p, dm, pts)
    sdf_or, dep_or = oracle_query(p, dm, pts)
    assert_parity(sdf, dep, sdf_or, dep_or, TOL_BF16)


@pytest.mark.parametrize("H", [16, 32, 64, 128, 256, 336])
@pytest.mark.parametrize("tail", [0, 1])
def test_fp32_random_depths_small(H, tail):
    L = 4
    spec = g.TMlpSpec(L=L, H=H, omega0=30.0, tail=tail, seed=5)
    p = g.make_weights(spec)
    dm = _random_voxel_map(4, L, 3)
    pts = _pts(5003, 4)
    with make_ctx(spec, FP32) as ctx:
        sdf, dep = run_engine(ctx, p, dm, pts)
    sdf_or, dep_or = oracle_query(p, dm, pts)
    assert_parity(sdf, dep, sdf_or, dep_or, TOL_FP32)


def test_fp32_wide_deep_net():
    """SAND_FP32 with an 8x256 net (the register-blocked FP32 query kernel for wide nets): all depths
    1..8 over many binned 128-row tiles (two 64-point sub-tiles each) with ragged ends, 1e-4 parity."""
    spec = g.TMlpSpec(L=8, H=256, omega0=30.0, tail=0, seed=17)
    p = g.make_weights(spec)
    dm = _random_voxel_map(4, 8, 5)
    pts = _pts(40011, 6)
    with make_ctx(spec, FP32) as ctx:
        sdf, dep = run_engine(ctx, p, dm, pts)
    sdf_or, dep_or = oracle_query(p, dm, pts)
    assert_parity(sdf, dep, sdf_or, dep_or, TOL_FP32)


def test_C0_full_fp32():
    """BASELINE.json configs[0] at full size (262,144 points), every point vs the oracle."""
    c = g.make_config("C0")
    p = c.params()
    pts = c.points_fn()
    with make_ctx(c.spec, FP32) as ctx:
        sdf, dep = run_engine(ctx, p, c.depthmap, pts)
        st = ctx.sand_get_stats()
    sdf_or, dep_or = oracle_query(p, c.depthmap, pts)
    assert_parity(sdf, dep, sdf_or, dep_or, TOL_FP32)
    assert sum(st["per_depth"]) + st["n_nonfinite"] == pts.shape[0]
    np.testing.assert_array_equal(st["per_depth"], np.bincount(dep_or, minlength=c.spec.L + 1))


def test_C1_full_bf16():
    """configs[1] (256^3 grid, 16.8M points): exit depth of every point bit-exact; SDF on a seeded
    uniform + per-depth stratified sample."""
    c = g.make_config("C1")
    p = c.params()
    pts = c.points_fn()
    with make_ctx(c.spec, BF16) as ctx:
        sdf, dep = run_engine(ctx, p, c.depthmap, pts)
    d_or, _, _ = oracle.lookup(c.depthmap, pts)
    np.testing.assert_array_equal(dep, d_or)
    idx = stratified_sample(dep, 4096, 1 << 16, seed=1)
    sdf_or, dep_or = oracle_query(p, c.depthmap, pts[idx])
    assert_parity(sdf, dep, sdf_or, dep_or, TOL_BF16, idx=idx)


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_C2_C3_full_size_sampled(name):
    """configs[2] (512^3 grid, 134M points, level-7 octree) and configs[3] (8x336, 8M cloud) in the
    bench's launch configuration: exit depths of all points bit-exact, SDF on a stratified
    sample."""
    c = g.make_config(name)
    p = c.params()
    pts = c.points_fn()
    with make_ctx(c.spec, BF16) as ctx:
        sdf, dep = run_engine(ctx, p, c.depthmap, pts)
        st = ctx.sand_get_stats()
    n = pts.shape[0]
    # exit depths of every point, oracle lookup slab by slab (bounded host memory)
    step = 1 << 24
    for q0 in range(0, n, step):
        d_or, _, _ = oracle.lookup(c.depthmap, pts[q0:q0 + step])
        np.testing.assert_array_equal(dep[q0:q0 + step], d_or)
    idx = stratified_sample(dep, 4096, 1 << 15, seed=2)
    sdf_or, dep_or = oracle_query(p, c.depthmap, pts[idx])
    assert_parity(sdf, dep, sdf_or, dep_or, TOL_BF16, idx=idx)
    assert sum(st["per_depth"]) + st["n_nonfinite"] == n
    assert st["per_depth"][0] == 0   # BJ configs have no far leaves


@pytest.mark.parametrize("prec,H", [(BF16, 64), (FP32, 32)])
def test_far_field_and_lod_caps(prec, H):
    """Eq. 7 depth-0 cached values; LOD cap 1..L (Sec. 3.4) incl. cap = L no-op."""
    L = 4
    spec = g.TMlpSpec(L=L, H=H, omega0=30.0, seed=6)
    p = g.make_weights(spec)
    dm = _random_voxel_map(3, L, 7, far=True)
    pts = _pts(3000, 8)
    tol = TOL_BF16 if prec == BF16 else TOL_FP32
    with make_ctx(spec, prec) as ctx:
        for cap in (1, 2, 3, L):
            sdf, dep = run_engine(ctx, p, dm, pts, cap=cap)
            sdf_or, dep_or = oracle_query(p, dm, pts, lod_cap=cap)
            assert_parity(sdf, dep, sdf_or, dep_or, tol)
    far = dep_or == 0
    assert far.any()
    np.testing.assert_array_equal(sdf[far], sdf_or[far].astype(np.float32))


def test_octree_descent_and_baked_paths():
    """Octree levels 9 and 10 (device descent, no baking) and level 6 (baked dense grid), far-field
    leaves included; out-of-domain and face points."""
    L = 6
    spec = g.TMlpSpec(L=L, H=64, omega0=30.0, seed=9)
    p = g.make_weights(spec)
    sph = g.make_spheres(3, n=4)
    rng = np.random.default_rng(0)
    pts = np.concatenate([rng.uniform(-1.2, 1.2, (20000, 3)),
                          -1 + rng.integers(0, 513, (2000, 3)) * (2.0 / 512)]).astype(np.float32)
    for lev in (6, 9, 10):
        oc = g.build_octree(sph, lev, g.configs.BANDS_8, L, score_seed=1, far_band=True,
                            subdivide_factor=0.3)
        with make_ctx(spec, BF16) as ctx:
            sdf, dep = run_engine(ctx, p, oc, pts)
        sdf_or, dep_or = oracle_query(p, oc, pts)
        assert_parity(sdf, dep, sdf_or, dep_or, TOL_BF16)


def test_nonfinite_and_edge_sizes():
    """NaN/Inf points -> depth 255, sdf NaN; n in {0, 1, 3, 129}; unaligned (4-byte) point buffer."""
    import torch
    L = 3
    spec = g.TMlpSpec(L=L, H=64, omega0=30.0, seed=10)
    p = g.make_weights(spec)
    dm = _random_voxel_map(2, L, 11)
    base = _pts(200, 12)
    base[5] = [np.nan, 0, 0]
    base[17] = [0, np.inf, 0]
    base[18] = [0, 0, -np.inf]
    with make_ctx(spec, BF16) as ctx:
        ctx.sand_load_weights(g.pack_blob(p))
        ctx.sand_load_depthmap(dm)
        for n in (0, 1, 3, 129, 200):
            pts = base[:n]
            sdf_or, dep_or = oracle_query(p, dm, pts)
            sdf, dep = run_engine(ctx, p, dm, pts) if n else (np.zeros(0, np.float32), np.zeros(0, np.uint8))
            if n:
                assert_parity(sdf, dep, sdf_or, dep_or, TOL_BF16)
        # unaligned: points start 1 float into the buffer (4-byte but not 16-byte aligned)
        flat = torch.from_numpy(np.concatenate([[0.0], base.ravel()]).astype(np.float32)).cuda()
        sdf_t = torch.empty(200, dtype=torch.float32, device="cuda")
        dep_t = torch.empty(201, dtype=torch.uint8, device="cuda")
        ctx.sand_set_stream(torch.cuda.current_stream().cuda_stream)
        ctx.sand_query(flat.data_ptr() + 4, 200, sdf_t.data_ptr(), dep_t.data_ptr() + 1)
        torch.cuda.synchronize()
        sdf_or, dep_or = oracle_query(p, dm, base)
        assert_parity(sdf_t.cpu().numpy(), dep_t.cpu().numpy()[1:], sdf_or, dep_or, TOL_BF16)


def test_binning_is_stable_depth_partition():
    """K2 (S:412 depth-bucketed batching): perm is a permutation of the near points, grouped by
    depth deepest-first, ascending point order within a depth (stable)."""
    L = 6
    spec = g.TMlpSpec(L=L, H=64, omega0=30.0, seed=12)
    p = g.make_weights(spec)
    dm = _random_voxel_map(3, L, 13, far=True)
    pts = _pts(50001, 14)
    with make_ctx(spec, BF16) as ctx:
        _, dep = run_engine(ctx, p, dm, pts)
        perm = ctx.sand_debug_perm()
    _, dep_or = oracle_query(p, dm, pts)
    expect = np.concatenate([np.nonzero(dep_or == d)[0] for d in range(L, 0, -1)])
    np.testing.assert_array_equal(perm, expect.astype(np.uint32))


def test_determinism_and_host_e2e():
    """Two runs bit-identical; sand_query_host (chunked, pinned host buffers) equals sand_query."""
    import torch
    c = g.make_config("C1")
    p = c.params()
    pts = c.points_fn(0, 64)   # first 64 z-planes of the 256^3 grid
    with make_ctx(c.spec, BF16) as ctx:
        s1, d1 = run_engine(ctx, p, c.depthmap, pts)
        s2, d2 = run_engine(ctx, p, c.depthmap, pts)
        np.testing.assert_array_equal(s1, s2)
        np.testing.assert_array_equal(d1, d2)
        n = pts.shape[0]
        hp = torch.from_numpy(pts).pin_memory()
        hs = torch.empty(n, dtype=torch.float32).pin_memory()
        hd = torch.empty(n, dtype=torch.uint8).pin_memory()
        for chunk in (1 << 20, 0, 12345):   # explicit, library default, ragged chunks
            hs.zero_()
            hd.zero_()
            ctx.sand_query_host(hp.data_ptr(), n, hs.data_ptr(), hd.data_ptr(), chunk_points=chunk)
            np.testing.assert_array_equal(hs.numpy(), s1)
            np.testing.assert_array_equal(hd.numpy(), d1)


def test_shard_invariance_of_the_multi_gpu_partition():
    """SURVEY 8(e) pin: the z-slab shards of partition.shard_planes (world = 1, 2, 4, 8), each queried on
    its own as a rank would, reproduce the single-query SDF and exit depths bit for bit (per-point math
    does not depend on tile mates)."""
    import torch
    from paper_2604_25936_b200 import partition
    c = g.make_config("C1")
    p = c.params()
    R = c.grid_R
    pts = g.grid_points(R)
    with make_ctx(c.spec, BF16) as ctx:
        s_all, d_all = run_engine(ctx, p, c.depthmap, pts)
        for world in (2, 4, 8):
            s_sh = np.empty_like(s_all)
            d_sh = np.empty_like(d_all)
            for rank in range(world):
                k0, k1, _ = partition.shard_planes(c.depthmap, R, world, rank, weak=False)
                sl = slice(k0 * R * R, k1 * R * R)
                sdf, dep = ctx.query_tensor(torch.from_numpy(np.ascontiguousarray(pts[sl])).cuda())
                torch.cuda.synchronize()
                s_sh[sl], d_sh[sl] = sdf.cpu().numpy(), dep.cpu().numpy()
            np.testing.assert_array_equal(d_sh, d_all)
            np.testing.assert_array_equal(s_sh, s_all)


def test_all_max_depth_equals_full_depth():
    """BJ oracle check 2 on the GPU: an all-L map == uniform full-depth evaluation (query_full)."""
    L = 8
    spec = g.TMlpSpec(L=L, H=256, omega0=30.0, seed=15)
    p = g.make_weights(spec)
    dm = g.VoxelMap(1, np.full(8, L, np.uint8), None)
    pts = _pts(20000, 16)
    with make_ctx(spec, BF16) as ctx:
        sdf, dep = run_engine(ctx, p, dm, pts)
    assert (dep == L).all()
    full = oracle.query_full(p, pts)
    assert np.abs(sdf - full).max() <= TOL_BF16


@pytest.mark.parametrize("L,tail", [(20, 0), (32, 0), (32, 1)])
def test_deep_nets_pair_kernel_limits(L, tail):
    """Deep T-MLPs at H = 256.  With w0 and the biases folded into the MMA operands the CTA-pair kernel's
    on-chip tables are the tail vectors only, so L = 32 LINEAR fits it and must match the oracle; a
    configuration that fits no BF16 kernel (L = 32 MULT keeps two tail vectors per layer) must either
    match as well or be refused cleanly with SAND_ERR_UNSUPPORTED (include/sand.h), never mis-computed."""
    from paper_2604_25936_b200 import SandError
    spec = g.TMlpSpec(L=L, H=256, omega0=30.0, tail=tail, seed=21)
    try:
        ctx = make_ctx(spec, BF16)
    except SandError as e:
        assert tail == 1 and e.code == -7
        return
    p = g.make_weights(spec)
    dm = _random_voxel_map(3, L, 22)
    pts = _pts(6001, 23)
    with ctx:
        sdf, dep = run_engine(ctx, p, dm, pts)
    sdf_or, dep_or = oracle_query(p, dm, pts)
    assert_parity(sdf, dep, sdf_or, dep_or, TOL_BF16)


def test_options_explicit_and_pair_kernel_switch():
    """sand_set_option (no environment variables): defaults, bad keys / values, and every kernel selectable
    through SAND_OPT_PAIR_KERNEL (2 = slot-team CTA-pair, 1 = two-pass CTA-pair, 0 = 1-CTA) gives the same
    exit depths and SDF within the BF16 tolerance on the same context."""
    from paper_2604_25936_b200 import SAND_OPT_DYN_SCHEDULE, SAND_OPT_KPROF, SAND_OPT_PAIR_KERNEL, SandError
    spec = g.TMlpSpec(L=5, H=256, omega0=30.0, seed=77)
    p = g.make_weights(spec)
    rng = np.random.default_rng(8)
    dm = g.VoxelMap(4, rng.integers(1, 6, 4096).astype(np.uint8), None)
    pts = rng.uniform(-1, 1, (70001, 3)).astype(np.float32)
    sdf_or, dep_or = oracle_query(p, dm, pts)
    with make_ctx(spec, BF16) as ctx:
        assert ctx.sand_get_option(SAND_OPT_PAIR_KERNEL) == 2
        assert ctx.sand_get_option(SAND_OPT_DYN_SCHEDULE) == 0
        assert ctx.sand_get_option(SAND_OPT_KPROF) == 0
        for bad in ((99, 0), (SAND_OPT_PAIR_KERNEL, 3), (SAND_OPT_PAIR_KERNEL, -1), (SAND_OPT_DYN_SCHEDULE, -1),
                    (SAND_OPT_KPROF, 7)):
            with pytest.raises(SandError):
                ctx.sand_set_option(*bad)
        res = {}
        for mode in (2, 1, 0):
            ctx.sand_set_option(SAND_OPT_PAIR_KERNEL, mode)
            assert ctx.sand_get_option(SAND_OPT_PAIR_KERNEL) == mode
            res[mode] = run_engine(ctx, p, dm, pts)
    for mode in (2, 1, 0):
        assert_parity(*res[mode], sdf_or, dep_or, TOL_BF16)


@pytest.mark.parametrize("L", [1, 2, 3])
@pytest.mark.parametrize("H", [64, 128, 256])
def test_bf16_shallow_nets_team_kernel(L, H):
    """The slot-team kernel (SAND_OPT_PAIR_KERNEL 2) at its protocol edges: L = 1 (no hidden layer: no weight image,
    every job a layer-1 job), L = 2 (one hidden layer: every owner job followed by a sharer), L = 3; odd tile counts
    per depth (the scan pads each bin to an even count of 256-row tiles) and a ragged last tile."""
    from paper_2604_25936_b200 import SAND_OPT_PAIR_KERNEL
    spec = g.TMlpSpec(L=L, H=H, omega0=30.0, tail=0, seed=120 + 7 * L + H)
    p = g.make_weights(spec)
    dm = _random_voxel_map(3, L, 121 + L)
    pts = _pts(3 * 256 * L + 77, 122 + L)
    sdf_or, dep_or = oracle_query(p, dm, pts)
    with make_ctx(spec, BF16) as ctx:
        assert ctx.sand_get_option(SAND_OPT_PAIR_KERNEL) == 2
        sdf, dep = run_engine(ctx, p, dm, pts)
    assert_parity(sdf, dep, sdf_or, dep_or, TOL_BF16)


@pytest.mark.parametrize("H", [64, 128, 256])
@pytest.mark.parametrize("tail", [0, 1])
@pytest.mark.parametrize("mode", [1, 2])
def test_bf16_pair_kernels_both(H, tail, mode):
    """Both CTA-pair kernels (SAND_OPT_PAIR_KERNEL 1: two N-half passes per layer, 16 lock-step epilogue warps;
    2: one N = H chain per layer, one epilogue team per tile slot, weight stages shared by the slots) on every
    depth 1..L, many 256-row tiles per depth with ragged tails, and a second query on the same context (the
    persistent kernels' barrier phases restart per launch)."""
    from paper_2604_25936_b200 import SAND_OPT_PAIR_KERNEL
    L = 8
    spec = g.TMlpSpec(L=L, H=H, omega0=30.0, tail=tail, seed=90 + H + tail)
    p = g.make_weights(spec)
    dm = _random_voxel_map(4, L, 91)
    pts = _pts(150001, 92)
    sdf_or, dep_or = oracle_query(p, dm, pts)
    with make_ctx(spec, BF16) as ctx:
        ctx.sand_set_option(SAND_OPT_PAIR_KERNEL, mode)
        for _ in range(2):
            sdf, dep = run_engine(ctx, p, dm, pts)
            assert_parity(sdf, dep, sdf_or, dep_or, TOL_BF16)


@pytest.mark.parametrize("name", [
    "C1",
    pytest.param("C2", marks=pytest.mark.skipif(os.environ.get("SAND_FULL_PARITY") != "1",
                                                reason="opt-in (SAND_FULL_PARITY=1): 134M points on the CPU oracle")),
    pytest.param("C3", marks=pytest.mark.skipif(os.environ.get("SAND_FULL_PARITY") != "1",
                                                reason="opt-in (SAND_FULL_PARITY=1)")),
])
def test_full_sdf_all_points(name):
    """SDF of EVERY point of configs[1..3] against the FP32 C oracle (OpenMP on the host
    cores).  C1 (16.8M points) runs in the default suite; C2 / C3 are opt-in (their default tests sample)."""
    c = g.make_config(name)
    p = c.params()
    pts = c.points_fn()
    with make_ctx(c.spec, BF16) as ctx:
        sdf, dep = run_engine(ctx, p, c.depthmap, pts)
    step = 1 << 22
    for q0 in range(0, pts.shape[0], step):
        idx = np.arange(q0, min(q0 + step, pts.shape[0]))
        sdf_or, dep_or = oracle_query(p, c.depthmap, pts[idx])
        assert_parity(sdf, dep, sdf_or, dep_or, TOL_BF16, idx=idx)


@pytest.mark.parametrize("H", [64, 128, 256])
@pytest.mark.parametrize("tail", [0, 1])
def test_f16x3_random_depths(H, tail):
    """SAND_F16X3 (split-FP16 three-product MMAs, FP32 accuracy): mixed depths 1..L with ragged tiles at the
    FP32 tolerance 1e-4 against the FP32 C oracle."""
    from paper_2604_25936_b200 import SAND_F16X3
    L = 6
    spec = g.TMlpSpec(L=L, H=H, omega0=30.0, tail=tail, seed=70 + H)
    p = g.make_weights(spec)
    dm = _random_voxel_map(3, L, 71)
    pts = _pts(30011, 72)
    pts[17] = [np.nan, 0, 0]
    with make_ctx(spec, SAND_F16X3) as ctx:
        sdf, dep = run_engine(ctx, p, dm, pts)
    sdf_or, dep_or = oracle_query(p, dm, pts)
    assert_parity(sdf, dep, sdf_or, dep_or, TOL_FP32)


def test_f16x3_c0_full_and_c2_sample():
    """BASELINE.json configs[0] (the FP32 config) on the split-FP16 tensor path, every point; and C2's 8 x 256 net
    on a stratified sample of its grid, both at the FP32 tolerance."""
    from paper_2604_25936_b200 import SAND_F16X3
    c = g.make_config("C0")
    p = c.params()
    pts = c.points_fn()
    with make_ctx(c.spec, SAND_F16X3) as ctx:
        sdf, dep = run_engine(ctx, p, c.depthmap, pts)
    sdf_or, dep_or = oracle_query(p, c.depthmap, pts)
    assert_parity(sdf, dep, sdf_or, dep_or, TOL_FP32)
    c = g.make_config("C2")
    p = c.params()
    pts = g.grid_points_slab(512, 240, 272)
    with make_ctx(c.spec, SAND_F16X3) as ctx:
        sdf, dep = run_engine(ctx, p, c.depthmap, pts)
    idx = stratified_sample(dep, 4096, 1 << 15, seed=3)
    sdf_or, dep_or = oracle_query(p, c.depthmap, pts[idx])
    assert_parity(sdf, dep, sdf_or, dep_or, TOL_FP32, idx=idx)
