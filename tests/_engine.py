"""Test helpers: run seeded inputs through libsand (via the Python binding) and through the oracle."""
import numpy as np

import sandgen as g

TOL_BF16 = 5e-3   # BASELINE.json north_star: BF16 path max-abs
TOL_FP32 = 1e-4   # BASELINE.json north_star: FP32/TF32 path max-abs
SIGN_EPS = 5e-3   # sign must agree wherever |f_oracle| > 5e-3


def oracle_query(params, depthmap, points, lod_cap=None):
    """The GPU parity reference: the plain FP32 C oracle (oracle/sand_oracle_fp32.c, BASELINE.json's
    north-star oracle; pinned against the float64 numpy oracle by tests/test_oracle_fp32.py).  Returns
    (sdf float64 [n], exit depth u8 [n]) like oracle.query."""
    from oracle import fp32
    sdf, dep = fp32.query_fp32(params, depthmap, points, lod_cap=lod_cap)
    return sdf.astype(np.float64), dep


def make_ctx(spec, precision, device=0):
    from paper_2604_25936_b200 import SandContext
    return SandContext(spec.L, spec.H, spec.omega0, precision, spec.tail, device)


def run_engine(ctx, params, depthmap, pts_np, cap=None):
    import torch
    ctx.sand_load_weights(g.pack_blob(params))
    ctx.sand_load_depthmap(depthmap)
    if cap is not None:
        ctx.sand_set_lod_cap(cap)
    pts = torch.from_numpy(np.ascontiguousarray(pts_np, np.float32)).cuda()
    sdf, dep = ctx.query_tensor(pts)
    torch.cuda.synchronize()
    return sdf.cpu().numpy(), dep.cpu().numpy()


def assert_parity(sdf_gpu, dep_gpu, sdf_or, dep_or, tol, idx=None):
    """Exit depth bit-exact; SDF max-abs <= tol; sign agreement where |oracle| > SIGN_EPS;
    non-finite points NaN on both sides."""
    if idx is not None:
        sdf_gpu, dep_gpu = sdf_gpu[idx], dep_gpu[idx]
    np.testing.assert_array_equal(dep_gpu, dep_or)
    nan_or = np.isnan(sdf_or)
    assert np.array_equal(np.isnan(sdf_gpu), nan_or), "NaN pattern differs"
    ok = ~nan_or
    err = np.abs(sdf_gpu[ok].astype(np.float64) - sdf_or[ok])
    mx = float(err.max()) if err.size else 0.0
    assert mx <= tol, f"max-abs error {mx:.3e} > {tol:.1e} (at {int(np.argmax(err))})"
    big = np.abs(sdf_or[ok]) > SIGN_EPS
    assert np.array_equal(np.sign(sdf_gpu[ok][big]), np.sign(sdf_or[ok][big])), "sign mismatch"
    return mx


def stratified_sample(dep, per_depth, n_uniform, seed=0):
    """Seeded subset: n_uniform uniform indices + up to per_depth indices of every exit depth."""
    rng = np.random.default_rng(seed)
    n = dep.size
    parts = [rng.choice(n, size=min(n_uniform, n), replace=False)]
    for d in np.unique(dep):
        w = np.nonzero(dep == d)[0]
        parts.append(rng.choice(w, size=min(per_depth, w.size), replace=False))
    return np.unique(np.concatenate(parts))
