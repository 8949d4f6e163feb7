#!/bin/bash
# Build a libsand variant with extra defines for tmlp_tc2.cu into abl/libsand_<name>.so
# usage: scripts/variant.sh <name> "<defines>"   (ALLDEFS="..." adds defines to every source)
cd "$(dirname "$0")/.." || exit 1
mkdir -p abl
C=paper_2604_25936_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I include"
objs=""
for src in sand_api lookup tmlp_simt tmlp_tc tmlp_tc3 depthpop mesh; do
  nvcc $F ${ALLDEFS} -c $C/$src.cu -o abl/$src.o & objs="$objs abl/$src.o"
done
nvcc $F $2 -c $C/tmlp_tc2.cu -o abl/tc2_$1.o &
wait
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o abl/libsand_$1.so $objs abl/tc2_$1.o -cudart static
rm -f abl/*.o
ls -la abl/libsand_$1.so
