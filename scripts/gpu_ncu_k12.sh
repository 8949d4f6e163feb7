#!/bin/bash
# K1 / K2b: one ncu --set full capture each (C2, after warm-up) + the launch list of one bench step
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-full-depth"
$CMD > gpurun_out/ncu12_plain.log 2>&1 && \
ncu --kernel-name regex:"k_lookup|k_scatter" --launch-skip 4 --launch-count 2 --set full --import-source on --clock-control none -o gpurun_out/k12_prof -f $CMD > gpurun_out/k12_ncu.log 2>&1; echo "ncu rc=$?"
python scripts/ncu_rows.py gpurun_out/k12_prof.ncu-rep > gpurun_out/k12_summary.txt 2>&1; cat gpurun_out/k12_summary.txt
