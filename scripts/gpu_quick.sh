# quick: a subset of parity tests + kprof + bench (np variants)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bf16_random or binning or nonfinite or far_field or all_max or determinism" > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/q_pytest.log
SAND_KPROF=1 timeout 120 python bench.py --no-cpu --no-e2e --steps 1 2>&1 | grep kprof | tail -1
for np in ${NPOLYS:-4}; do
  SAND_NPOLY=$np timeout 120 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/q_bench_np$np.log 2>&1; echo "bench np=$np rc=$?"
  python -c "
import json
l=[x for x in open('gpurun_out/q_bench_np$np.log') if x.startswith('{')]
if l:
  d=json.loads(l[-1]); print('np=$np value %.3e ms %.2f mlp %.2f frac %.3f' % (d['value'], d['ms_per_step'], d['stage_ms']['mlp'], d['roofline']['frac']))
else: print(open('gpurun_out/q_bench_np$np.log').read()[-2000:])
"
done
