cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -k 10 780 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fv_tests.log 2>&1
echo "tests rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/fv_tests.log | tail -8
timeout -k 10 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout -k 10 200 python bench.py > gpurun_out/fv_bench.json 2> gpurun_out/fv_bench.err
tail -1 gpurun_out/fv_bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', round(d['ms_per_step'],1), round(d['value']), round(d['e2e']['value']), d['roofline']['frac'], d['clocks'])" || tail -5 gpurun_out/fv_bench.err
