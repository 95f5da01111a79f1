# Round-2 launch lists with DRAM traffic (1 x B200): every launch of one timed step (after 3 warm-ups) of the
# C3 (1.3B) and C2 (GPT-2-small) workloads: duration + dram read / write bytes per launch.  Plain runs first.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/r2b_c3.json 2> gpurun_out/r2b_c3.err || exit 1
python bench.py --workload gpt2s --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_c2.json 2> gpurun_out/r2b_c2.err || exit 1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none -c 4000 --csv --log-file gpurun_out/r2b_launches_c3.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2b_ncu_c3.log 2>&1
ncu --metrics $M --clock-control none -c 6000 --csv --log-file gpurun_out/r2b_launches_c2.csv \
    python bench.py --workload gpt2s --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2b_ncu_c2.log 2>&1
tail -n 2 gpurun_out/r2b_ncu_c3.log gpurun_out/r2b_ncu_c2.log
