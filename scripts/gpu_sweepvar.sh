#!/bin/bash
# uniform-depth sweep (DEPTHS) for each abl/libsand_<name>.so
for name in "$@"; do SAND_LIB=abl/libsand_$name.so timeout 300 python scripts/depth_sweep.py 2>&1 | grep "ns/step"; done
