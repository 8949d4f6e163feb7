"""Debug: per-depth / per-feature-range error of the CTA-pair kernel against the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle
import sandgen as g
from _engine import make_ctx, run_engine
H = int(sys.argv[1]) if len(sys.argv) > 1 else 256
for L in (1, 2, 3):
    for d in range(1, L + 1):
        spec = g.TMlpSpec(L=L, H=H, omega0=30.0, tail=0, seed=4)
        p = g.make_weights(spec)
        dm = g.VoxelMap(1, np.full(8, d, np.uint8), None)
        pts = np.random.default_rng(2).uniform(-1, 1, (3000, 3)).astype(np.float32)
        with make_ctx(spec, 2) as ctx:
            sdf, dep = run_engine(ctx, p, dm, pts)
        sdf_or, dep_or = oracle.query(p, dm, pts)
        err = np.abs(sdf - sdf_or)
        print(f"H={H} L={L} d={d}: depth ok {np.array_equal(dep, dep_or)} maxabs {err.max():.3e} rows>tol {(err > 5e-3).sum()} "
              f"first bad rows {np.nonzero(err > 5e-3)[0][:8]}")
