# peer-memory DP: parity + path evidence on 2 GPUs, then C3 A/B peer vs NCCL at 2 GPUs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -k 10 900 python -m pytest tests/test_gpu_dist.py -x -q -k "dp2 or dp_" -p no:cacheprovider > gpurun_out/dpc_tests.log 2>&1
echo "tests rc=$?"; tail -25 gpurun_out/dpc_tests.log
run() {  # gpus name args
  timeout -k 10 420 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) \
    bench.py --gpus $1 --steps 4 --warmup 3 --no-e2e $3 > gpurun_out/dpc_$2.json 2> gpurun_out/dpc_$2.err
  tail -1 gpurun_out/dpc_$2.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['comm_last_step_rank0']
print('$2', round(d['ms_per_step'],1), round(d['value']), 'exposed', round(d['exposed_comm_ms_per_step'],2), d['gpu_launches'], d['clocks']['sm_mhz'])" || tail -6 gpurun_out/dpc_$2.err
}
run 2 peer2 ""
run 2 nccl2 "--nccl-dp"
run 2 peer2b ""
