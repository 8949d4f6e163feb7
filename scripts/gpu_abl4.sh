for v in base a1 a2 a4 a8 a10 a15; do SAND_LIB=abl/libsand_$v.so DEPTHS=1,2,8 timeout 200 python scripts/depth_sweep.py 2>&1 | grep -v Warn; done
R=1 bash scripts/gpu_ab4.sh abl base a1 a2 a4 a8 a10 a15
