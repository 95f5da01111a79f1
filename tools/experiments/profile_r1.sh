# Launch list of one 1.3B step (ncu, serialised, cold L2: compare shares), plus a plain bench run first.
cd $GRAFT_REPO_ROOT
python bench.py --steps 5 --warmup 3 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 1900 -c 1100 --csv --log-file gpurun_out/launches_r1_final.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
tail -1 gpurun_out/ncu_launch.log
