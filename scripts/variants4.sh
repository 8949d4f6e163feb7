#!/bin/bash
# Build libsand variants differing only in tmlp_tc4.cu defines into abl/libsand_<name>.so.
# usage: scripts/variants4.sh "name1:-DA=1 -DB=2" "name2:-DC=3" ...
cd "$(dirname "$0")/.." || exit 1
mkdir -p abl/obj4
C=paper_2604_25936_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I include"
objs=""
for src in sand_api lookup tmlp_simt tmlp_tc tmlp_tc2 tmlp_tc3 tmlp_x3 depthpop mesh; do
  nvcc $F ${ALLDEFS} -c $C/$src.cu -o abl/obj4/$src.o & objs="$objs abl/obj4/$src.o"
done
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  nvcc $F ${ALLDEFS} $defs -c $C/tmlp_tc4.cu -o abl/obj4/tc4_$name.o &
done
wait
for spec in "$@"; do
  name=${spec%%:*}
  nvcc -shared -gencode arch=compute_100a,code=sm_100a -o abl/libsand_$name.so $objs abl/obj4/tc4_$name.o -cudart static
done
rm -rf abl/obj4
ls -la abl/*.so
