# kernel + step parity tests, default bench, launch list of one C3 step (durations + DRAM bytes)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_hbm_kernels.py tests/test_gpu_step.py tests/test_gpu_post_ln.py tests/test_gpu_guard.py -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err || exit 1
python - <<'PY'
import json
j = json.loads(open("gpurun_out/r2k_bench.json").read().strip().splitlines()[-1])
print(j["ms_per_step"], j["value"], j["kernels"]["attention"], j["clocks"]["sm_mhz"])
PY
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none -c 4000 --csv --log-file gpurun_out/r2k_launches_c3.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2k_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/r2k_launches_c3.csv --last 749 | head -24
