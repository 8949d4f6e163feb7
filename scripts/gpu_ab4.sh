#!/bin/bash
# Interleaved A/B of abl/libsand_<name>.so variants on C2 (R rounds; power-cap noise needs interleaving).
# usage: R=2 scripts/gpu_ab4.sh tag name1 name2 ...
tag=$1; shift
mkdir -p gpurun_out
for r in $(seq 1 ${R:-2}); do
for name in "$@"; do
  SAND_LIB=abl/libsand_$name.so timeout ${VAR_TIMEOUT:-200} python bench.py --no-cpu --no-e2e --no-full-depth --steps ${STEPS:-20} ${BENCH_ARGS} > gpurun_out/${tag}_${name}_$r.log 2>&1
  python - "$tag" "$name" "$r" <<'PY'
import json, sys
tag, name, r = sys.argv[1:4]
l = [x for x in open(f'gpurun_out/{tag}_{name}_{r}.log') if x.startswith('{')]
if l:
    d = json.loads(l[-1]); c = d.get('clocks') or {}
    print('%-8s r%s value %.3e ms %.2f mlp %.2f frac %.3f sm %s W %s sum %s' % (name, r, d['value'], d['ms_per_step'], d['stage_ms']['mlp'], d['roofline']['frac'], c.get('sm_mhz'), c.get('power_w_median'), d['checksums']['sdf_fixed_point_2^24']))
else:
    print(name, open(f'gpurun_out/{tag}_{name}_{r}.log').read()[-1500:])
PY
done
done
