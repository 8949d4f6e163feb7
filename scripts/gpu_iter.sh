# usage: bash scripts/gpu_iter.sh <tag> [pytest-args]  -- parity tests, then bench variants (no ncu)
tag=${1:-it}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/${tag}_pytest.log
for np in ${NPOLYS:-4}; do
  SAND_NPOLY=$np timeout 300 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/${tag}_bench_np$np.log 2>&1; echo "bench np=$np rc=$?"
  python -c "
import json,sys
l=[x for x in open('gpurun_out/${tag}_bench_np$np.log') if x.startswith('{')]
if l:
  d=json.loads(l[-1]); print('np=$np value %.3e ms %.2f mlp %.2f frac %.3f' % (d['value'], d['ms_per_step'], d['stage_ms']['mlp'], d['roofline']['frac']))
else: print(open('gpurun_out/${tag}_bench_np$np.log').read()[-2000:])
"
done
