# wide kernel (H = 336) check: parity subset + C3 bench (+ kprof)
mkdir -p gpurun_out
if [ -z "$NOTEST" ]; then
timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "336 or wide or C3" > gpurun_out/t3_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t3_pytest.log
fi
SAND_KPROF=1 timeout 120 python bench.py --config C3 --no-cpu --no-e2e --steps 1 --warmup 1 2>&1 | grep kprof3 | tail -1
timeout 200 python bench.py --config C3 --no-cpu --no-e2e --steps 10 > gpurun_out/t3_bench.log 2>&1; echo "bench rc=$?"
python -c "
import json
l=[x for x in open('gpurun_out/t3_bench.log') if x.startswith('{')]
d=json.loads(l[-1]); print('value %.3e ms %.2f mlp %.3f frac %.4f' % (d['value'], d['ms_per_step'], d['stage_ms']['mlp'], d['roofline']['frac']))
" || tail -c 1500 gpurun_out/t3_bench.log
