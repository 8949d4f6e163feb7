"""GPU parity for the dynamic-exit query without a depth map ('SAND w/o Octree', PAPER.md P:736-738;
DESIGN.md reading R23) through the C ABI (sand_query_dynamic) against oracle.query_dynamic.

The exit layer is a threshold decision |t_i| < r taken in FP32 on the GPU and in float64 by the oracle:
points whose residual sits within FP32 evaluation error of r may legitimately stop one layer apart.  For
those the test checks that the GPU's layer is valid under the rule with that slack and that its SDF is
the oracle's y at the GPU's layer; every other point must match exactly (layer) and within 1e-4 (SDF)."""
import numpy as np
import pytest

import oracle
import sandgen as g
from _engine import make_ctx
from paper_2604_25936_b200 import SAND_OPT_DYN_SCHEDULE

pytestmark = pytest.mark.gpu
EPS = 2e-5   # FP32 evaluation error budget of t_i / y_i on these nets (accurate sinf, L <= 8)
FP32, BF16 = 0, 2


def _run(ctx, pts, r):
    import torch
    n = pts.shape[0]
    t = torch.from_numpy(np.ascontiguousarray(pts)).cuda()
    sdf = torch.empty(n, dtype=torch.float32, device="cuda")
    dep = torch.empty(n, dtype=torch.uint8, device="cuda")
    ctx.sand_set_stream(torch.cuda.current_stream().cuda_stream)
    ctx.sand_query_dynamic(t.data_ptr(), n, r, sdf.data_ptr(), dep.data_ptr())
    torch.cuda.synchronize()
    return sdf.cpu().numpy(), dep.cpu().numpy()


def _check(p, pts, r, sdf, dep):
    sdf_or, dep_or = oracle.query_dynamic(p, pts, r)
    fin = dep_or != oracle.NONFINITE_DEPTH
    np.testing.assert_array_equal(dep[~fin], dep_or[~fin])
    assert np.all(np.isnan(sdf[~fin]))
    _, ts, ys = oracle.tmlp_trace(p, pts[fin])
    L = p.spec.L
    d, do = dep[fin].astype(np.int64), dep_or[fin].astype(np.int64)
    # validity of the GPU layer under the rule with slack EPS
    ok = np.ones(d.size, bool)
    for i in range(2, L):
        at, before = d == i, d > i
        ok &= ~at | (np.abs(ts[i - 1]) < r + EPS)
        ok &= ~before | (np.abs(ts[i - 1]) >= r - EPS)
    assert ok.all(), f"{(~ok).sum()} invalid exit layers"
    same = d == do
    assert same.mean() >= 0.99, f"only {same.mean():.4f} of exit layers match"
    y_at = ys[d - 1, np.arange(d.size)]
    np.testing.assert_allclose(sdf[fin], y_at, rtol=0, atol=1e-4)
    return same.mean(), np.bincount(d, minlength=L + 1)


@pytest.mark.parametrize("pool", [0, 1, 2])
@pytest.mark.parametrize("H,L,tail", [(64, 6, 0), (256, 8, 0), (128, 5, 1), (336, 8, 0), (32, 1, 0), (64, 1, 0)])
def test_dynamic_exit_matches_oracle(H, L, tail, pool):
    """Schedules 0 / 1: FP32 SIMT tile exit / re-compaction; 2: all layers on the split-FP16 tensor kernel with
    the exit selected afterwards (H in {64, 128, 256}; other widths must be refused)."""
    spec = g.TMlpSpec(L=L, H=H, omega0=30.0, tail=tail, seed=21 + H)
    p = g.make_weights(spec)
    pts = np.random.default_rng(H).uniform(-1, 1, (5003, 3)).astype(np.float32)
    pts[7] = [np.nan, 0, 0]
    pts[100] = [0, np.inf, 0]
    if L > 1:
        _, ts, _ = oracle.tmlp_trace(p, pts[:2000][np.isfinite(pts[:2000]).all(1)])
        r = float(np.quantile(np.abs(ts[1:]), 0.3))   # about 30% of residuals below r: exits spread
    else:
        r = 1.0
    with make_ctx(spec, BF16 if H >= 64 else FP32) as ctx:   # the dynamic path is FP32 in either context
        ctx.sand_set_option(SAND_OPT_DYN_SCHEDULE, pool)   # tile-level exit / re-compaction / tensor select
        ctx.sand_load_weights(g.pack_blob(p))
        if pool == 2 and H not in (64, 128, 256):
            from paper_2604_25936_b200 import SandError
            with pytest.raises(SandError) as e:
                _run(ctx, pts, r)
            assert e.value.code == -7
            return
        sdf, dep = _run(ctx, pts, r)
    frac, hist = _check(p, pts, r, sdf, dep)
    if L > 2:
        assert hist[2] > 0 and hist[L] > 0, hist   # some points stop early, some run to L


@pytest.mark.parametrize("pool", [0, 1, 2])
def test_dynamic_special_cases_and_sizes(pool):
    """r = 0 -> full depth (= query_full); huge r -> everyone stops at layer 2; n in {0, 1, 65} and a
    ragged last tile."""
    spec = g.TMlpSpec(L=5, H=64, omega0=30.0, seed=31)
    p = g.make_weights(spec)
    pts = np.random.default_rng(3).uniform(-1, 1, (1000, 3)).astype(np.float32)
    with make_ctx(spec, FP32) as ctx:
        ctx.sand_set_option(SAND_OPT_DYN_SCHEDULE, pool)
        assert ctx.sand_get_option(SAND_OPT_DYN_SCHEDULE) == pool
        ctx.sand_load_weights(g.pack_blob(p))
        sdf, dep = _run(ctx, pts, 0.0)
        assert np.all(dep == 5)
        np.testing.assert_allclose(sdf, oracle.query_full(p, pts), rtol=0, atol=1e-4)
        sdf, dep = _run(ctx, pts, 1e30)
        assert np.all(dep == 2)
        np.testing.assert_allclose(sdf, oracle.tmlp_forward(p, pts, 2), rtol=0, atol=1e-4)
        for n in (1, 65):
            sdf, dep = _run(ctx, pts[:n], 0.0)
            assert np.all(dep == 5)
        import torch
        z = torch.zeros(1, device="cuda")
        ctx.sand_query_dynamic(z.data_ptr(), 0, 0.5, z.data_ptr(), z.data_ptr())   # n = 0: no-op
        with pytest.raises(Exception):
            ctx.sand_query_dynamic(z.data_ptr(), 4, -1.0, z.data_ptr(), z.data_ptr())
