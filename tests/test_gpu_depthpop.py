"""GPU parity for depth-map population (Sec. 3.2, Eq. 5 and Eq. 6) through the C ABI
(sand_required_depth, sand_populate_leaf_depths) against the oracle.

Eq. 5 turns floating point into an integer (a threshold on |y_L - y_i| and a sign test).  The kernel
decides in FP32 (R22), the oracle in float64, so points whose deciding quantities sit within
FP32 evaluation error of the threshold (or of zero, for the sign) may legitimately differ: for those
the test checks that the GPU's depth is a valid answer under the rule with that slack; every other
point must match exactly, and at least 99% of points must match."""
import numpy as np
import pytest

import oracle
import sandgen as g

pytestmark = pytest.mark.gpu
EPS = 2e-5   # FP32 evaluation error budget of y_i on these nets (|y| ~ 0.1, L <= 8, accurate sinf)


def _valid(ys, d, r, near):
    """GPU depth d (1-based) is valid under Eq. 5 with slack EPS (ys: oracle float64 [L][n])."""
    L, n = ys.shape
    yL = ys[-1]
    ok = np.ones(n, bool)
    for i in range(1, L + 1):
        yi = ys[i - 1]
        sign_amb = (np.abs(yi) < EPS) | (np.abs(yL) < EPS)
        same = (np.sign(yi) == np.sign(yL)) | sign_amb
        diff_sign = (np.sign(yi) != np.sign(yL)) | sign_amb
        close = np.abs(yL - yi) < r + EPS if near else np.ones(n, bool)
        far = np.abs(yL - yi) >= r - EPS if near else np.zeros(n, bool)
        at = d == i
        ok &= ~at | (same & close) | (i == L)            # the chosen i satisfies the rule (i = L always)
        before = d > i
        ok &= ~before | diff_sign | far                    # every earlier i may fail it
    return ok


def _run_required(ctx, pts, r, near):
    import torch
    t = torch.from_numpy(pts).cuda()
    out = torch.empty(pts.shape[0], dtype=torch.uint8, device="cuda")
    ctx.sand_set_stream(torch.cuda.current_stream().cuda_stream)
    ctx.sand_required_depth(t.data_ptr(), pts.shape[0], r, near, out.data_ptr())
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.int64)


@pytest.mark.parametrize("tensor", [1, 0])
@pytest.mark.parametrize("H,L,tail,prec", [(16, 4, 0, 0), (64, 6, 1, 0), (256, 8, 0, 2), (256, 8, 1, 2),
                                           (336, 8, 0, 2), (128, 5, 0, 2), (64, 1, 0, 2)])
@pytest.mark.parametrize("near", [True, False])
def test_required_depth_matches_oracle(H, L, tail, prec, near, tensor):
    """tensor = 1: H in {64, 128, 256} on the split-FP16 tensor-core kernel (tmlp_x3.cu); 0: FP32 SIMT."""
    from paper_2604_25936_b200 import SAND_OPT_FP32_TENSOR, SandContext
    spec = g.TMlpSpec(L=L, H=H, omega0=30.0, tail=tail, seed=41)
    p = g.make_weights(spec)
    pts = np.random.default_rng(42).uniform(-1, 1, (20011, 3)).astype(np.float32)
    _, _, ys = oracle.tmlp_trace(p, pts)
    r = float(np.quantile(np.abs(ys[-1] - ys[L // 2]), 0.5)) if L > 1 else 1e-3   # spreads the decisions over 1..L
    d_or = oracle.required_depth(p, pts, r, near=near)
    with SandContext(L, H, 30.0, prec, tail, 0) as ctx:
        ctx.sand_set_option(SAND_OPT_FP32_TENSOR, tensor)
        ctx.sand_load_weights(g.pack_blob(p))
        d = _run_required(ctx, pts, r, near)
    assert d.min() >= 1 and d.max() <= L
    mism = d != d_or
    assert mism.mean() < 0.01, f"{mism.mean():.4f} of points differ"
    assert np.all(_valid(ys[:, mism], d[mism], r, near)), "GPU depth invalid under Eq. 5 at differing points"
    if near and L > 1:
        assert len(np.unique(d_or)) > 1   # the threshold really decides something


@pytest.mark.parametrize("tensor", [1, 0])
def test_populate_leaf_depths_c2_octree_leaves(tensor):
    """Eq. 6 on the C2 octree's finest leaves with the paper's r = 1.5e-4 and a loose r."""
    import torch
    from paper_2604_25936_b200 import SAND_OPT_FP32_TENSOR, SandContext
    c = g.make_config("C2")
    p = c.params()
    oc = c.depthmap
    sel = np.nonzero(oc.leaf_level == oc.level)[0][:1500]
    samples = g.leaf_samples(oc.leaf_level[sel], oc.leaf_ijk[sel], 16, seed=5)   # 25 per leaf
    n, spl = samples.shape[0], samples.shape[1]
    with SandContext(c.spec.L, c.spec.H, 30.0, 2, 0, 0) as ctx:
        ctx.sand_set_option(SAND_OPT_FP32_TENSOR, tensor)
        ctx.sand_load_weights(g.pack_blob(p))
        ts = torch.from_numpy(np.ascontiguousarray(samples.reshape(-1, 3))).cuda()
        for r in (1.5e-4, 0.05):
            out = torch.empty(n, dtype=torch.uint8, device="cuda")
            ctx.sand_set_stream(torch.cuda.current_stream().cuda_stream)
            ctx.sand_populate_leaf_depths(ts.data_ptr(), n, spl, r, out.data_ptr())
            per = _run_required(ctx, samples.reshape(-1, 3), r, True).reshape(n, spl)
            torch.cuda.synchronize()
            got = out.cpu().numpy().astype(np.int64)
            np.testing.assert_array_equal(got, per.max(axis=1))          # pooling of the GPU's own d(x)
            exp = oracle.populate_leaf_depths(p, samples, r)
            mism = got != exp
            assert mism.mean() < 0.02
            if mism.any():   # differing leaves: some sample of theirs is near-threshold
                _, _, ys = oracle.tmlp_trace(p, samples[mism].reshape(-1, 3))
                assert np.all(_valid(ys, per[mism].reshape(-1), r, True))


def test_populate_edge_sizes():
    import torch
    from paper_2604_25936_b200 import SandContext
    spec = g.TMlpSpec(L=3, H=64, omega0=30.0, seed=43)
    p = g.make_weights(spec)
    with SandContext(3, 64, 30.0, 2, 0, 0) as ctx:
        ctx.sand_load_weights(g.pack_blob(p))
        ctx.sand_populate_leaf_depths(0, 0, 1, 1e-3, 0)     # n_leaves = 0: no-op
        pts = np.random.default_rng(44).uniform(-1, 1, (7, 1, 3)).astype(np.float32)
        t = torch.from_numpy(pts.reshape(-1, 3)).cuda()
        out = torch.empty(7, dtype=torch.uint8, device="cuda")
        ctx.sand_set_stream(torch.cuda.current_stream().cuda_stream)
        ctx.sand_populate_leaf_depths(t.data_ptr(), 7, 1, 1e-3, out.data_ptr())
        torch.cuda.synchronize()
        exp = oracle.populate_leaf_depths(p, pts, 1e-3)
        assert np.mean(out.cpu().numpy() == exp) >= 6 / 7


def test_leaf_max_pooling_hand_case_gpu():
    """SPEC S:304 / Eq. 6 on the GPU: the hand-built net of tests/test_oracle_depthpop.py (padded to H = 16 with
    zero units) gives per-sample depths {1, 3, 2} and the leaf depth 3."""
    import torch
    from paper_2604_25936_b200 import SandContext
    from test_oracle_depthpop import HAND_D, hand_pool_net, hand_pool_samples
    p = hand_pool_net(H=16)
    s = hand_pool_samples()
    with SandContext(3, 16, 1.0, 0, 0, 0) as ctx:
        ctx.sand_load_weights(g.pack_blob(p))
        d = _run_required(ctx, s, 0.05, True)
        np.testing.assert_array_equal(d, HAND_D)
        t = torch.from_numpy(np.ascontiguousarray(s)).cuda()
        out = torch.empty(1, dtype=torch.uint8, device="cuda")
        ctx.sand_populate_leaf_depths(t.data_ptr(), 1, 3, 0.05, out.data_ptr())
        torch.cuda.synchronize()
        assert int(out.item()) == 3
