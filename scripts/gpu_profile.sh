# usage: bash scripts/gpu_profile.sh <tag>   -- full GPU tests, bench lines, launch list, ncu --set full of K3
tag=${1:-v8}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${tag}_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/${tag}_bench_c2.log 2>&1; echo "bench c2 rc=$?"
timeout 300 python bench.py --config C3 > gpurun_out/${tag}_bench_c3.log 2>&1; echo "bench c3 rc=$?"
timeout 300 python bench.py --config C1 --no-cpu > gpurun_out/${tag}_bench_c1.log 2>&1; echo "bench c1 rc=$?"
timeout 300 python bench.py --full-depth --no-cpu --no-e2e > gpurun_out/${tag}_bench_c2_full.log 2>&1; echo "bench full rc=$?"
timeout 300 python bench.py --task populate > gpurun_out/${tag}_bench_pop.log 2>&1; echo "bench pop rc=$?"
timeout 600 python bench.py --task sweep --steps 5 > gpurun_out/${tag}_bench_sweep.log 2>&1; echo "bench sweep rc=$?"
timeout 600 python bench.py --task dynamic > gpurun_out/${tag}_bench_dynamic.log 2>&1; echo "bench dynamic rc=$?"
timeout 600 python bench.py --task mesh > gpurun_out/${tag}_bench_mesh.log 2>&1; echo "bench mesh rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${tag}_bench_ref.log 2>&1; echo "bench ref rc=$?"
python bench.py --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/${tag}_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/${tag}_ncu1.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tmlp -s 2 -c 1 -o gpurun_out/${tag}_prof_tc2 python bench.py --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/${tag}_ncu2.log 2>&1
echo "ncu tc2 rc=$?"
python bench.py --config C3 --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/${tag}_plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tmlp_wide -s 2 -c 1 -o gpurun_out/${tag}_prof_tc3 python bench.py --config C3 --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/${tag}_ncu3.log 2>&1
echo "ncu tc3 rc=$?"
