"""bench.py's N > 1 path (torchrun, one process per GPU, z-slab weak scaling, per-rank record gather,
max-over-ranks timing), run with 2 ranks sharing the visible GPU (SAND_BENCH_SHARE_GPU=1: gloo instead of
NCCL).  The ranks' kernels never wait on each other, so sharing one GPU is safe."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_weak_scaling_line():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--no-cpu", "--no-e2e", "--config", "C1"]
    r = subprocess.run(cmd, cwd=ROOT, env=dict(os.environ, SAND_BENCH_SHARE_GPU="1"), capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, "exactly one JSON line (rank 0)"
    d = lines[0]
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    assert d["config"]["global_points"] == 2 * 256 ** 3          # 256 x 256 x 512 grid
    assert sum(d["per_depth"]) == d["config"]["global_points"]   # every point binned once
    assert d["value"] > 0 and d["roofline"]["frac"] > 0
