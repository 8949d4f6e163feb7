"""Time sand_marching_cubes alone on a 512^3 analytic sdf grid (sphere union) -- profiling helper."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import sandgen as g
from paper_2604_25936_b200 import SandContext

R = int(sys.argv[1]) if len(sys.argv) > 1 else 512
ax = torch.tensor((2.0 * np.arange(R) / (R - 1) - 1.0).astype(np.float32), device="cuda")
Z, Y, X = torch.meshgrid(ax, ax, ax, indexing="ij")
sph = g.make_spheres(g.configs.SPHERE_SEED)
sdf = torch.full((R, R, R), 1e9, device="cuda")
for c, r in zip(sph.centres, sph.radii):
    sdf = torch.minimum(sdf, torch.sqrt((X - float(c[0])) ** 2 + (Y - float(c[1])) ** 2 + (Z - float(c[2])) ** 2) - float(r))
sdf = sdf.contiguous()
with SandContext(2, 64, 30.0, 2, 0, 0) as ctx:
    n = ctx.sand_marching_cubes(sdf.data_ptr(), R, 0, 0)
    tris = torch.empty(9 * n, device="cuda")
    for _ in range(3):
        ctx.sand_marching_cubes(sdf.data_ptr(), R, tris.data_ptr(), n)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ctx.sand_marching_cubes(sdf.data_ptr(), R, tris.data_ptr(), n)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"R {R}: {n} triangles, {ms:.3f} ms per call, {(4 * R**3 + 36 * n) / ms / 1e6:.0f} GB/s algorithmic")
