# N1 A/B on one box: C3 data parallelism over peer memory (default) vs NCCL, at 2 and 4 GPUs, twice each
cd $GRAFT_REPO_ROOT
run() {  # gpus name args
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) \
    bench.py --gpus $1 --steps 4 --warmup 3 --no-e2e $3 > gpurun_out/dp_$2.json 2> gpurun_out/dp_$2.err
  tail -1 gpurun_out/dp_$2.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['comm_last_step_rank0']
print('$2', round(d['ms_per_step'],1), round(d['value']), 'exposed', round(d['exposed_comm_ms_per_step'],2), 'ag', c['ag_bytes'], 'rs', c['rs_bytes'], d['clocks']['sm_mhz'])" || tail -4 gpurun_out/dp_$2.err
}
for rep in 1 2; do
  run 4 peer4_$rep ""
  run 4 nccl4_$rep "--nccl-dp"
done
run 2 peer2 ""
run 2 nccl2 "--nccl-dp"
python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('one_gpu', round(d['ms_per_step'],1), round(d['value']), d['clocks']['sm_mhz'])"
