cd $GRAFT_REPO_ROOT
timeout 300 python tools/parity_report.py r1 > gpurun_out/parity.log 2>&1
timeout 200 python bench.py --workload gpt2s --steps 4 --warmup 3 > gpurun_out/bench_gpt2s.json 2> gpurun_out/bench_gpt2s.err
timeout 200 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 1950 -c 1000 --csv --log-file gpurun_out/launches_r1b.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
echo done
