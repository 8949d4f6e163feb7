"""Tiny adaptive query through the C ABI for compute-sanitizer runs (tier T4)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import sandgen as g  # noqa: E402
from paper_2604_25936_b200 import SAND_BF16, SAND_FP32, SandContext  # noqa: E402

rng = np.random.default_rng(0)
pts = torch.from_numpy(rng.uniform(-1, 1, (3001, 3)).astype(np.float32)).cuda()
for prec, H, L in ((SAND_BF16, 256, 4), (SAND_BF16, 64, 3), (SAND_FP32, 32, 3)):
    spec = g.TMlpSpec(L=L, H=H, omega0=30.0, seed=1)
    p = g.make_weights(spec)
    dm = g.VoxelMap(2, rng.integers(0 if prec == SAND_FP32 else 1, L + 1, 64).astype(np.uint8),
                    rng.normal(size=64).astype(np.float32))
    with SandContext(L, H, 30.0, prec, 0, 0) as ctx:
        ctx.sand_load_weights(g.pack_blob(p))
        ctx.sand_load_depthmap(dm)
        sdf, dep = ctx.query_tensor(pts)
        torch.cuda.synchronize()
        print("ok", prec, H, float(sdf.abs().max()))
