# full bench line (default C2) + other configs + launch list for profiles/
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_c2.log 2>&1; echo "c2 rc=$?"
for c in C1 C3; do python bench.py --config $c --no-cpu --steps 5 > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; done
python bench.py --full-depth --no-cpu --no-e2e --steps 3 > gpurun_out/bench_c2_full.log 2>&1; echo "full rc=$?"
python bench.py --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v7.csv python bench.py --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/ncu_l.log 2>&1; echo "ncu rc=$?"
