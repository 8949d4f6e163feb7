"""K3 time per step for uniform depth maps d = 1..8 on C2's grid and net (the shallow vs deep regimes)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import sandgen as g
from paper_2604_25936_b200 import SAND_BF16, SandContext

c = g.make_config("C2")
p = c.params()
pts = torch.from_numpy(g.grid_points_slab(512, 0, 256)).cuda()   # 67M points
n = pts.shape[0]
sdf = torch.empty(n, device="cuda")
dep = torch.empty(n, dtype=torch.uint8, device="cuda")
out = {}
with SandContext(8, 256, 30.0, SAND_BF16, 0, 0) as ctx:
    ctx.sand_load_weights(g.pack_blob(p))
    ctx.sand_reserve(n)
    ctx.sand_set_stream(torch.cuda.current_stream().cuda_stream)
    if os.environ.get("PK"):
        from paper_2604_25936_b200 import SAND_OPT_PAIR_KERNEL
        ctx.sand_set_option(SAND_OPT_PAIR_KERNEL, int(os.environ["PK"]))
    for d in [int(v) for v in os.environ.get("DEPTHS", "1,2,3,4,8").split(",")]:
        ctx.sand_load_depthmap(g.VoxelMap(1, np.full(8, d, np.uint8), None))
        for _ in range(3):
            ctx.sand_query(pts.data_ptr(), n, sdf.data_ptr(), dep.data_ptr())
        ctx.sand_get_stats()
        for _ in range(5):
            ctx.sand_query(pts.data_ptr(), n, sdf.data_ptr(), dep.data_ptr())
        st = ctx.sand_get_stats()
        ms = st["ms_mlp_sum"] / st["queries"]
        steps_per_pair = n / 256 * d / 74
        out[d] = {"ms_k3": ms, "ns_per_step_per_pair": ms * 1e6 / steps_per_pair,
                  "tensor_frac": n * (d - 1) * 2 * 256 * 256 / (ms / 1e3) / 1648.6e12}
        print(os.environ.get("SAND_LIB", "in-tree"), d, "%.1f ns/step/pair  tensor %.3f" % (out[d]["ns_per_step_per_pair"], out[d]["tensor_frac"]), flush=True)
json.dump(out, open("gpurun_out/depth_sweep_%s.json" % os.path.basename(os.environ.get("SAND_LIB", "intree")), "w"))
