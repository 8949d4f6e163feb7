#!/bin/bash
TAG=r02_v8
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/${TAG}_c2.json 2> gpurun_out/${TAG}_c2.err; echo "bench rc=$?"
tail -c 600 gpurun_out/${TAG}_c2.json
