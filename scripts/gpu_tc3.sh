# wide kernel (H = 336) check: parity subset + C3 bench
mkdir -p gpurun_out
SAND_HANG_TIMEOUT=1 timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "336 or wide or C3" > gpurun_out/t3_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/t3_pytest.log
timeout 200 python bench.py --config C3 --no-cpu --no-e2e --steps 10 > gpurun_out/t3_bench.log 2>&1; echo "bench rc=$?"; tail -c 1500 gpurun_out/t3_bench.log
