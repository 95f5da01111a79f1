# C2 (GPT-2-small) on the current build: bench + launch list with DRAM bytes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --workload gpt2s --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2n_c2.json 2> gpurun_out/r2n_c2.err || exit 1
python -c "import json; j=json.loads(open('gpurun_out/r2n_c2.json').read().strip().splitlines()[-1]); print(j['ms_per_step'], j['value'], j['clocks']['sm_mhz'], j['e2e']['value'] if j.get('e2e') else None, j['roofline']['frac'])"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none -c 6000 --csv --log-file gpurun_out/r2n_launches_c2.csv \
    python bench.py --workload gpt2s --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2n_ncu.log 2>&1
tail -1 gpurun_out/r2n_ncu.log | cut -c1-200
