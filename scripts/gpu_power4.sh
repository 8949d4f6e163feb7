#!/bin/bash
# C2 (40 steps) and C4 (4 steps) time / clock / power for abl/libsand_<name>.so variants
for name in "$@"; do
  for cfg in C2 C4; do
    st=40; [ $cfg = C4 ] && st=4
    SAND_LIB=abl/libsand_$name.so timeout 150 python bench.py --config $cfg --no-cpu --no-e2e --no-full-depth --steps $st > gpurun_out/p4_${name}_$cfg.log 2>&1
    grep -h '^{' gpurun_out/p4_${name}_$cfg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['clocks']; print('%-10s %s %8.2f ms frac %.3f sm %s W %s' % ('$name', '$cfg', d['stage_ms']['mlp'], d['roofline']['frac'], c['sm_mhz'], c.get('power_w_median')))"
  done
done
