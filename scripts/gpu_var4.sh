#!/bin/bash
# A/B timing of abl/libsand_<name>.so variants on C2 with the slot-team kernel: usage gpu_var4.sh tag name1 name2 ...
tag=$1; shift
mkdir -p gpurun_out
for name in "$@"; do
  SAND_LIB=abl/libsand_$name.so timeout ${VAR_TIMEOUT:-200} python bench.py --no-cpu --no-e2e --no-full-depth --steps 10 --pair-kernel ${PK:-2} ${BENCH_ARGS} > gpurun_out/${tag}_$name.log 2>&1
  python - "$tag" "$name" <<'PY'
import json, sys
tag, name = sys.argv[1], sys.argv[2]
l = [x for x in open(f'gpurun_out/{tag}_{name}.log') if x.startswith('{')]
if l:
    d = json.loads(l[-1]); c = d.get('clocks') or {}
    print('%-8s value %.3e ms %.2f mlp %.2f frac %.3f sm %s' % (name, d['value'], d['ms_per_step'], d['stage_ms']['mlp'], d['roofline']['frac'], c.get('sm_mhz')))
else:
    print(name, open(f'gpurun_out/{tag}_{name}.log').read()[-1500:])
PY
done
