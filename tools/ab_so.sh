# A/B of two library builds on one box: default bench (5 steps) alternated, then the launch list (DRAM bytes) of B
#   bash tools/ab_so.sh A B   (exp/A.so exp/B.so)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cp paper_2106_02679_b200/liblga.so /tmp/rel.so
for rep in 1 2; do for v in "$1" "$2"; do
  cp exp/$v.so paper_2106_02679_b200/liblga.so
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$v.json 2>/dev/null
  python -c "import json; j=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]); print('$v', round(j['ms_per_step'],2), round(j['value']), j['clocks']['sm_mhz'], round(j['roofline']['achieved']), round(j['kernels']['attention']['achieved_tflops']))"
done; done
cp exp/$2.so paper_2106_02679_b200/liblga.so
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none -c 4000 --csv --log-file gpurun_out/ab_launches_$2.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/gemm_traffic.py gpurun_out/ab_launches_$2.csv 1.3b 749
python tools/launch_summary.py gpurun_out/ab_launches_$2.csv --last 749 | head -8
cp /tmp/rel.so paper_2106_02679_b200/liblga.so
