# Round-2 closing run of the final build (1 x B200): full GPU suite, default bench, the launch list of one
# C3 step with per-launch DRAM bytes, then ncu --set full of the attention-backward kernels (dK/dV storing
# dS^T, dQ from dS).  Each ncu command runs only after the same program exited 0 without ncu.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2c_pytest.log
python bench.py > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err || exit 1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2c_bench10.json 2> gpurun_out/r2c_bench10.err || exit 1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none -c 4000 --csv --log-file gpurun_out/r2c_launches_c3.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2c_ncu_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:dkdv_kernel|dq_from_ds" -s 12 -c 4 \
    -o gpurun_out/r2c_attnbwd python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r2c_ncu_attn.log 2>&1
tail -n 3 gpurun_out/r2c_pytest.log gpurun_out/r2c_ncu_c3.log gpurun_out/r2c_ncu_attn.log
cat gpurun_out/r2c_bench.json
