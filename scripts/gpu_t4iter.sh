#!/bin/bash
# slot-team kernel iteration: parity subset on the in-tree build, variant timings, uniform-depth sweep
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pair_kernels_both or options_explicit or bf16_random_depths_small" > gpurun_out/it_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/it_pytest.log
bash scripts/gpu_var4.sh it "$@"
SAND_LIB=abl/libsand_base.so timeout 300 python scripts/depth_sweep.py 2>&1 | tail -5
