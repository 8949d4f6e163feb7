#!/bin/bash
# Build ablation variants of libsand (SAND_ABL=1..4 in tmlp_tc2.cu; timing only, wrong results) into abl/.
# Use with SAND_LIB=abl/libsand_N.so python bench.py ...
cd "$(dirname "$0")/.." || exit 1
mkdir -p abl
C=paper_2604_25936_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I include"
objs=""
for src in sand_api lookup tmlp_simt tmlp_tc tmlp_tc3 depthpop mesh; do
  nvcc $F -c $C/$src.cu -o abl/$src.o & objs="$objs abl/$src.o"
done
for v in ${ABLS:-1 2 3 4}; do nvcc $F -DSAND_ABL=$v -c $C/tmlp_tc2.cu -o abl/tc2_$v.o & done
wait
for v in ${ABLS:-1 2 3 4}; do
  nvcc -shared -gencode arch=compute_100a,code=sm_100a -o abl/libsand_$v.so $objs abl/tc2_$v.o -cudart static
done
rm -f abl/*.o
ls -la abl/*.so
