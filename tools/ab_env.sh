# A/B of an environment setting on one box: bash tools/ab_env.sh "VAR=a" "VAR=b" ...  (C3 bench, alternated x2)
cd $GRAFT_REPO_ROOT
for rep in 1 2; do for v in "$@"; do
  env $v python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abenv.log 2>&1
  python -c "import json; j=json.loads(open('gpurun_out/abenv.log').read().strip().splitlines()[-1]); print('$v', round(j['ms_per_step'],1), round(j['value']), j['clocks']['sm_mhz'], round(j['kernels']['attention']['achieved_tflops']))"
done; done
