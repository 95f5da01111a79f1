# Round-2 4-GPU session 6 (final build): the multi-rank suite on 4 GPUs (incl. the NCCL baseline), C3 scaling
# 1 / 2 / 4 GPUs, the C4 pipeline (P = 4) with per-rank p2p waits.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -q -p no:cacheprovider 2>&1 | tail -3
run() {   # n out args...
  local n=$1 out=$2; shift 2
  if [ $n -eq 1 ]; then
    timeout 600 python bench.py --no-cpu-baseline "$@" > $out 2> $out.err
  else
    timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29700 + RANDOM % 200)) bench.py --gpus $n "$@" > $out 2> $out.err
  fi
  tail -1 $out | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; ab=d.get('exposed_comm_ab') or {}; print('$out', c['schedule'], 'N', c['n_micro'], 'chunk', c['chunk'], 'dp', c['dp'], 'pp', c['pp'], 'ms', round(d['ms_per_step'],1), 'tok/s', round(d['value']), 'stall', [round(x,2) for x in d.get('exposed_comm_ms_per_step_ranks',[])], 'ab', round(ab.get('exposed_comm_ms_per_step', float('nan')),2), 'p2p', [round(x,1) for x in d.get('p2p_wait_ms_per_step_ranks',[])], 'clk', d['clocks'] and d['clocks']['sm_mhz'])" || tail -3 $out.err
}
for n in 1 2 4; do run $n gpurun_out/m6_scale_$n.json --steps 10 --warmup 3; done
run 4 gpurun_out/m6_c4_p4.json --workload 10b --steps 3 --warmup 3 --no-e2e --no-ab
