# multi-GPU slowdown diagnosis on one 4-GPU box: default vs --no-comm vs --nccl-dp (and 1 GPU)
cd $GRAFT_REPO_ROOT
run() {
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) \
    bench.py --gpus $1 --steps 4 --warmup 3 --no-e2e $3 > gpurun_out/if_$2.json 2> gpurun_out/if_$2.err
  tail -1 gpurun_out/if_$2.json | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$2', round(d['ms_per_step'],1), round(d['value']), 'exposed', round(d['exposed_comm_ms_per_step'],2), 'gemm', round(d['roofline']['achieved']), 'attn', round(d['kernels']['attention']['achieved_tflops']), 'adam', d['kernels']['adamw'], d['clocks']['sm_mhz'])" || tail -4 gpurun_out/if_$2.err
}
run 4 default ""
run 4 nocomm "--no-comm"
run 4 nccl "--nccl-dp"
python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('one', round(d['ms_per_step'],1), 'gemm', round(d['roofline']['achieved']), 'attn', round(d['kernels']['attention']['achieved_tflops']), 'adam', d['kernels']['adamw'], d['clocks']['sm_mhz'])"
