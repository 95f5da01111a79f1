# A/B of two builds on one box: alternate bench runs (exp/<a>.so, exp/<b>.so), print ms/step and clocks
cd $GRAFT_REPO_ROOT
cp paper_2106_02679_b200/liblga.so /tmp/rel.so
for rep in 1 2; do for v in "$@"; do
  cp exp/$v.so paper_2106_02679_b200/liblga.so
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$v.log 2>&1
  python -c "import json; j=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]); print('$v', round(j['ms_per_step'],1), round(j['value']), j['clocks']['sm_mhz'])"
done; done
cp /tmp/rel.so paper_2106_02679_b200/liblga.so
