#!/bin/bash
# K3 (C2): launch list of one bench step + one ncu --set full capture (source-level) of the CTA-pair kernel
mkdir -p gpurun_out
TAG=${1:-k3}
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-full-depth"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ll.log 2>&1; echo "launch list rc=$?"
ncu --kernel-name regex:"k_tmlp_tc[24]" --launch-skip 3 --launch-count 1 --set full --import-source on --clock-control none -o gpurun_out/${TAG}_prof -f $CMD > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
python scripts/ncu_summary.py gpurun_out/${TAG}_prof.ncu-rep > gpurun_out/${TAG}_summary.txt 2>&1; cat gpurun_out/${TAG}_summary.txt | head -40
