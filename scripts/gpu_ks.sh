#!/bin/bash
# K-split publish bring-up: parity subset on the default build, then interleaved A/B of abl/ variants on C2
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ks_build.log 2>&1 || { echo build failed; tail gpurun_out/ks_build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "${TESTS:-pair_kernels_both or options_explicit or bf16_random_depths_small or shallow_nets or deep_nets or C1_full}" > gpurun_out/ks_pytest.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/ks_pytest.log
[ -n "$VARIANTS" ] && R=${R:-2} scripts/gpu_ab4.sh ks $VARIANTS
