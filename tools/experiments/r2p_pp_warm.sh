# pipeline warm-up A/B at C4 (P = 4 on 4 GPUs): multi-rank suite, then bench with / without LGA_NO_PP_WARM
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -q -p no:cacheprovider 2>&1 | tail -2
run() {   # out env...
  local out=$1; shift
  env "$@" timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --workload 10b --steps 3 --warmup 3 --no-e2e --no-ab > $out 2> $out.err
  tail -1 $out | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$out', round(d['ms_per_step'],1), round(d['value']), 'p2p', [round(x,1) for x in d.get('p2p_wait_ms_per_step_ranks',[])], 'clk', d['clocks']['sm_mhz'], 'sends', d['comm_last_step_rank0']['p2p_send_calls'])" || tail -3 $out.err
}
for rep in 1 2; do
  run gpurun_out/pw_warm_$rep.json LGA_NO_PP_WARM=0
  run gpurun_out/pw_nowarm_$rep.json LGA_NO_PP_WARM=1
done
