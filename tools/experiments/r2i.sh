# attention forward with epilogue warps: kernel + step parity tests, default bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py tests/test_gpu_post_ln.py -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err
python - <<'PY'
import json
j = json.loads(open("gpurun_out/r2i_bench.json").read().strip().splitlines()[-1])
print(j["ms_per_step"], j["value"], j["kernels"]["attention"], j["clocks"]["sm_mhz"], j["e2e"]["value"])
PY
