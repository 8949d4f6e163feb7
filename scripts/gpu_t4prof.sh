#!/bin/bash
# per-role counters of the slot-team kernel on C2 and on uniform depth maps (SAND_T4_PROF build)
SAND_LIB=abl/libsand_prof.so timeout 200 python bench.py --no-cpu --no-e2e --no-full-depth --steps 1 --warmup 1 --pair-kernel 2 2>&1 | grep t4prof | tail -1
for d in 1 8; do SAND_LIB=abl/libsand_prof.so DEPTHS=$d timeout 200 python scripts/depth_sweep.py 2>&1 | grep t4prof | tail -1; done
