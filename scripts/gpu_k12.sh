#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
python bench.py --task sweep --steps 5 --no-cpu > gpurun_out/k12_sweep.json 2> gpurun_out/k12_sweep.err; echo "sweep rc=$?"
python bench.py --steps 10 --no-cpu --no-e2e --no-full-depth > gpurun_out/k12_c2.json 2>&1; echo "c2 rc=$?"
timeout 600 ncu --kernel-name regex:"k_lookup|k_scatter" --launch-skip 12 --launch-count 2 --set full --clock-control none -o gpurun_out/k12_ncu -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-full-depth > gpurun_out/k12_ncu.log 2>&1; echo "ncu rc=$?"
python - <<'PY'
import json
for f in ("k12_sweep", "k12_c2"):
    l=[x for x in open(f"gpurun_out/{f}.json") if x.startswith('{')]
    d=json.loads(l[-1]) if l else {}
    if f == "k12_c2":
        print(f, d.get("value"), d.get("stage_ms"), d.get("hbm_lookup_gbs"))
    else:
        for e in d.get("entries", []):
            print(f, {k: e.get(k) for k in ("map", "value", "stage_ms", "k1_hbm_gbs", "k1_frac_hbm")})
PY
