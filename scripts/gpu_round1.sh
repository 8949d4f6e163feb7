set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -2 gpurun_out/bench.log
python bench.py --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/ncu1.log 2>&1
echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_tmlp -s 2 -c 1 -o gpurun_out/prof_tc2 python bench.py --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/ncu2.log 2>&1
echo "ncu2 rc=$?"
