#!/bin/bash
# per-role counters (SAND_T4_PROF builds) of variants on C2 and uniform depths: usage scripts/gpu_ksprof.sh name...
for n in "$@"; do
echo "== $n"
SAND_LIB=abl/libsand_$n.so timeout 200 python bench.py --no-cpu --no-e2e --no-full-depth --steps 1 --warmup 1 --pair-kernel 2 2>&1 | grep t4prof | tail -1
for d in ${DEPTHS_LIST:-1 2 8}; do SAND_LIB=abl/libsand_$n.so DEPTHS=$d timeout 200 python scripts/depth_sweep.py 2>&1 | grep "t4prof\|ns per" | tail -2; done
done
