#!/bin/bash
# clock / power under the bench loop for abl/libsand_<name>.so variants (40 steps)
for name in "$@"; do
  SAND_LIB=abl/libsand_$name.so timeout 300 python bench.py --no-cpu --no-e2e --no-full-depth --steps 40 > gpurun_out/pw_$name.log 2>&1
  grep -h '^{' gpurun_out/pw_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', '%.2f ms' % d['stage_ms']['mlp'], d['clocks'])"
done
