"""Fused mesh extraction time vs slab thickness on C2's 512^3 grid (sand_mesh_grid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import sandgen as g
from paper_2604_25936_b200 import SAND_BF16, SandContext

c = g.make_config("C2")
p = c.params()
R = c.grid_R
dev = torch.device("cuda", 0)
with SandContext(c.spec.L, c.spec.H, c.spec.omega0, SAND_BF16, c.spec.tail, 0) as ctx:
    ctx.sand_load_weights(g.pack_blob(p))
    ctx.sand_load_depthmap(c.depthmap)
    st = torch.cuda.current_stream(dev)
    ctx.sand_set_stream(st.cuda_stream)
    ntri = ctx.sand_mesh_grid(R, 0, 0, 0)
    tris = torch.empty(9 * ntri, dtype=torch.float32, device=dev)
    for slab in [int(v) for v in os.environ.get("SLABS", "32,64,128,256,511").split(",")]:
        for _ in range(2):
            ctx.sand_mesh_grid(R, slab, tris.data_ptr(), ntri)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        e0.record(st)
        for _ in range(5):
            n = ctx.sand_mesh_grid(R, slab, tris.data_ptr(), ntri)
        e1.record(st)
        torch.cuda.synchronize(dev)
        print("slab %4d: %.2f ms per mesh, %d triangles" % (slab, e0.elapsed_time(e1) / 5, n), flush=True)
