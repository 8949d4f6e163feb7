"""CPU oracle for SAND's adaptive T-MLP query path.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import, call or execute anything under ``oracle/``.  The product path
(``paper_2604_25936_b200``) never imports it and has no CPU fallback.

Two independent restatements of the paper (PAPER.md = arxiv 2604.25936):

* ``oracle/sand_oracle_fp32.c`` (front end ``oracle.fp32``): the plain, slow FP32 C oracle BASELINE.json's
  north star names -- IEEE binary32, sequential sums, no FMA contraction, glibc ``sinf``, OpenMP over
  points.  The GPU parity tests, ``smoke()`` and the bench's CPU baseline / reference arm use it.
* ``oracle/sand_oracle.py``: a numpy twin in float64 for the network (float32 only where the kernel's
  float32 arithmetic decides an integer: the depth-map cell index, reading R1), plus the
  Sec. 8(f) functions (Eq. 5/6 population, dynamic exit, marching cubes).  It pins the FP32 oracle
  (tests/test_oracle_fp32.py: <= 1e-5 max-abs, exit depths bit-exact).

Pins (tests/test_oracle_*.py, all ``-m "not gpu"``): plain-SIREN special case vs torch float64
library layers; hand-computed L=2/H=1 golden values (tests/golden/); zero-parameter net; prefix
consistency; NaN poisoning of unused layers; Appendix-A quadratic form; init bounds/moments;
octree descent vs brute-force leaf scan; grid-point cells vs the integer closed form.
Parity unpinned: nothing in this module.
"""
from .sand_oracle import (
    cell_coords, lookup_voxel, lookup_octree, lookup_bruteforce, lookup,
    tmlp_forward, tmlp_trace, query, query_full, NONFINITE_DEPTH, required_depth, populate_leaf_depths,
    query_dynamic, marching_cubes, mc_loops,
)

__all__ = [
    "cell_coords", "lookup_voxel", "lookup_octree", "lookup_bruteforce", "lookup",
    "tmlp_forward", "tmlp_trace", "query", "query_full", "NONFINITE_DEPTH", "required_depth",
    "populate_leaf_depths", "query_dynamic", "marching_cubes", "mc_loops",
]
