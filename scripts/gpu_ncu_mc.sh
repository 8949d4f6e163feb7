#!/bin/bash
# ncu --set full capture of the marching-cubes kernel (unfused call of the mesh bench task)
mkdir -p gpurun_out
TAG=${1:-mc}
CMD="python bench.py --task mesh --no-cpu --steps 1 --warmup 1"
ncu --kernel-name regex:"${KREGEX:-k_mc_emit}" --launch-skip ${SKIP:-0} --launch-count 1 --set full --import-source on --clock-control none -o gpurun_out/${TAG}_prof -f $CMD > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
python scripts/ncu_summary.py gpurun_out/${TAG}_prof.ncu-rep > gpurun_out/${TAG}_summary.txt 2>&1; head -60 gpurun_out/${TAG}_summary.txt
