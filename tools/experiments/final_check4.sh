# 4 GPUs: whole GPU suite (peer-memory DP now active, post-LN), x32 post-LN bench, C3 DP A/B at 4 GPUs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -k 10 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fc_tests.log 2>&1
echo "tests rc=$?"; tail -30 gpurun_out/fc_tests.log
timeout -k 10 300 python bench.py --workload x32 --post-ln --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/fc_x32_post.json 2> gpurun_out/fc_x32_post.err
tail -1 gpurun_out/fc_x32_post.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('x32_post', round(d['ms_per_step'],1), round(d['value']), d['clocks']['sm_mhz'])" || tail -5 gpurun_out/fc_x32_post.err
run() {  # gpus name args
  timeout -k 10 420 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) \
    bench.py --gpus $1 --steps 4 --warmup 3 --no-e2e $3 > gpurun_out/fc_$2.json 2> gpurun_out/fc_$2.err
  tail -1 gpurun_out/fc_$2.json | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$2', round(d['ms_per_step'],1), round(d['value']), 'exposed', round(d['exposed_comm_ms_per_step'],2), d['gpu_launches'], d['clocks']['sm_mhz'])" || tail -6 gpurun_out/fc_$2.err
}
run 4 peer4 ""
run 4 nccl4 "--nccl-dp"
run 4 peer4b ""
run 4 nccl4b "--nccl-dp"
