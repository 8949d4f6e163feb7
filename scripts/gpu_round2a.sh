#!/bin/bash
# bench surface check: C2 default (full line), reference arm, C0, C4 on 1 GPU, then the multi-rank and C4 tests
mkdir -p gpurun_out
python bench.py --steps 10 > gpurun_out/r2a_c2.json 2> gpurun_out/r2a_c2.err; echo "c2 rc=$?"
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2a_ref.json 2> gpurun_out/r2a_ref.err; echo "ref rc=$?"
python bench.py --config C0 --steps 10 > gpurun_out/r2a_c0.json 2> gpurun_out/r2a_c0.err; echo "c0 rc=$?"
python bench.py --config C4 --steps 3 --no-e2e > gpurun_out/r2a_c4.json 2> gpurun_out/r2a_c4.err; echo "c4 rc=$?"
timeout 1500 python -m pytest tests/test_bench_multirank.py tests/test_gpu_c4.py -m gpu -x -q > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2a_pytest.log
for f in c2 ref c0 c4; do tail -c 600 gpurun_out/r2a_$f.err; python -c "
import json,sys
l=[x for x in open('gpurun_out/r2a_$f.json') if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
print('$f', {k: d.get(k) for k in ('value','ms_per_step','n_gpus','scaling')}, 'frac', (d.get('roofline') or {}).get('frac'), 'full', (d.get('full_depth_speedup') or {}).get('speedup'), 'cpu', d.get('cpu_baseline'))
"; done
