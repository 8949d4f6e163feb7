#!/bin/bash
mkdir -p gpurun_out
python bench.py --task populate --steps 5 --no-cpu > gpurun_out/x3_pop.json 2> gpurun_out/x3_pop.err; echo "pop rc=$?"
python bench.py --prec f16x3 --steps 5 --no-cpu --no-e2e > gpurun_out/x3_c2.json 2> gpurun_out/x3_c2.err; echo "c2 x3 rc=$?"
python bench.py --config C0 --prec f16x3 --steps 10 --no-cpu --no-e2e > gpurun_out/x3_c0.json 2> gpurun_out/x3_c0.err; echo "c0 x3 rc=$?"
python bench.py --prec fp32 --steps 3 --no-cpu --no-e2e > gpurun_out/x3_c2fp32.json 2> gpurun_out/x3_c2fp32.err; echo "c2 fp32 rc=$?"
for f in pop c2 c0 c2fp32; do tail -c 400 gpurun_out/x3_$f.err; python -c "
import json
l=[x for x in open('gpurun_out/x3_$f.json') if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
print('$f', d.get('value'), d.get('ms_per_step'), 'roof', {k:(d.get('roofline') or {}).get(k) for k in ('achieved','frac','kernel')}, 'simt', d.get('fp32_simt'))
"; done
