#!/bin/bash
# slot-team kernel bring-up: parity subset, then C2 timing of both CTA-pair kernels
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t4_build.log 2>&1 || { echo build failed; tail gpurun_out/t4_build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pair_kernels_both or options_explicit or bf16_random_depths_small" > gpurun_out/t4_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/t4_pytest.log
for k in ${KERNELS:-1 2}; do
  timeout 200 python bench.py --no-cpu --no-e2e --no-full-depth --steps 10 --pair-kernel $k ${BENCH_ARGS} > gpurun_out/t4_bench_k$k.log 2>&1; echo "bench k=$k rc=$?"
  python - "$k" <<'PY'
import json, sys
k = sys.argv[1]
l = [x for x in open(f'gpurun_out/t4_bench_k{k}.log') if x.startswith('{')]
if l:
    d = json.loads(l[-1]); c = d.get('clocks') or {}
    print('k=%s value %.3e ms %.2f mlp %.2f frac %.3f sm %s' % (k, d['value'], d['ms_per_step'], d['stage_ms']['mlp'], d['roofline']['frac'], c.get('sm_mhz')))
else:
    print(open(f'gpurun_out/t4_bench_k{k}.log').read()[-2000:])
PY
done
