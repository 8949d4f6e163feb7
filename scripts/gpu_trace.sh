#!/bin/bash
# per-job timelines (SAND_T4_TRACE build) for uniform depth 1 and 8 and for C2
mkdir -p gpurun_out
for d in 1 8; do SAND_LIB=abl/libsand_trace.so DEPTHS=$d timeout 200 python scripts/depth_sweep.py > /dev/null 2>&1; cp gpurun_out/t4trace.txt gpurun_out/t4trace_d$d.txt; cp gpurun_out/t4iotrace.txt gpurun_out/t4iotrace_d$d.txt; cp gpurun_out/t4wtrace.txt gpurun_out/t4wtrace_d$d.txt; done
SAND_LIB=abl/libsand_trace.so timeout 200 python bench.py --no-cpu --no-e2e --no-full-depth --steps 1 --warmup 1 > /dev/null 2>&1; cp gpurun_out/t4trace.txt gpurun_out/t4trace_c2.txt; cp gpurun_out/t4wtrace.txt gpurun_out/t4wtrace_c2.txt
