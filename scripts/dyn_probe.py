import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import sandgen as g
from paper_2604_25936_b200 import SandContext, SAND_BF16
c = g.make_config("C2"); p = c.params()
n = 1 << 22
pts = torch.from_numpy(g.grid_points(c.grid_R)[:n].copy()).cuda()
sdf = torch.empty(n, device="cuda"); dep = torch.empty(n, dtype=torch.uint8, device="cuda")
with SandContext(c.spec.L, c.spec.H, c.spec.omega0, SAND_BF16, c.spec.tail, 0) as ctx:
    ctx.sand_load_weights(g.pack_blob(p))
    for mode in ("0", "1"):
        os.environ["SAND_DYN_POOL"] = mode
        ctx.sand_query_dynamic(pts.data_ptr(), n, 1.5e-4, sdf.data_ptr(), dep.data_ptr()); torch.cuda.synchronize()
        t = time.perf_counter(); ctx.sand_query_dynamic(pts.data_ptr(), n, 1.5e-4, sdf.data_ptr(), dep.data_ptr()); torch.cuda.synchronize()
        print("lib", os.environ.get("SAND_LIB", "-"), "pool", mode, f"{(time.perf_counter() - t) * 1e3:.1f} ms")
