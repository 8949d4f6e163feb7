#!/bin/bash
# last check of the round after the marching-cubes pass-B changes: whole GPU suite, smoke, C2 and mesh bench lines
TAG=r02_v11
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_c2.json 2> gpurun_out/${TAG}_c2.err; echo "bench rc=$?"
timeout 900 python bench.py --task mesh --steps 5 --no-cpu > gpurun_out/${TAG}_mesh.json 2> gpurun_out/${TAG}_mesh.err; echo "mesh rc=$?"
tail -c 400 gpurun_out/${TAG}_mesh.json
