cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -k 5 120 python tools/attn_err.py > gpurun_out/attn_err.log 2>&1
rc=$?; cat gpurun_out/attn_err.log; echo "attn_err rc=$rc"; [ $rc -ne 0 ] && exit 1
timeout -k 10 480 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_post_ln.py tests/test_gpu_step.py -q -p no:cacheprovider > gpurun_out/rc_tests.log 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/rc_tests.log
timeout -k 10 200 python bench.py --steps 5 --warmup 3 > gpurun_out/rc_bench.json 2> gpurun_out/rc_bench.err
tail -1 gpurun_out/rc_bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', round(d['ms_per_step'],1), round(d['value']), d['e2e']['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])" || tail -5 gpurun_out/rc_bench.err
