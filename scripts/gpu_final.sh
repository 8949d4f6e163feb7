#!/bin/bash
# Round-2 validation and measurement set: GPU tests, smoke, every bench task, K3 launch list + ncu.
TAG=${1:-r02_final}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/${TAG}_$name.json 2> gpurun_out/${TAG}_$name.err; echo "bench $name rc=$?"; }
run c2 --steps 20 --warmup 5
run ref --impl reference --steps 20 --warmup 5
run c0 --config C0 --steps 20
run c1 --config C1 --steps 20
run c3 --config C3 --steps 10
run c4 --config C4 --steps 5 --no-e2e
run c2_f16x3 --prec f16x3 --steps 5 --no-e2e
run populate --task populate --steps 5
run sweep --task sweep --steps 5 --no-cpu
run dynamic --task dynamic --steps 3
run mesh --task mesh --steps 5 --no-cpu
bash scripts/gpu_ncu_k3.sh ${TAG}_k3
