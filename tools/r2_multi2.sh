# Round-2 multi-GPU follow-ups on one 4-GPU box:
#  1. C4 (10B) modular pipeline P = 4 x D = 1, chunk 4 and 8 (chunk 1, 2 in r2_multi.sh)
#  2. config-5 STANDARD step-time gap decomposed: STANDARD vs LAYERED at D = 1 (no communication), N = 16
#  3. STANDARD at D = 4, N = 16 with the no-comm A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() {   # n out args...
  local n=$1 out=$2; shift 2
  if [ $n -eq 1 ]; then
    timeout 600 python bench.py --no-cpu-baseline "$@" > $out 2> $out.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29700 + RANDOM % 200)) bench.py --gpus $n "$@" > $out 2> $out.err
  fi
  tail -1 $out | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; ab=d.get('exposed_comm_ab') or {}; print('$out', c['schedule'], 'N', c['n_micro'], 'chunk', c['chunk'], 'dp', c['dp'], 'pp', c['pp'], 'ms', round(d['ms_per_step'],1), 'tok/s', round(d['value']), 'stall', [round(x,2) for x in d.get('exposed_comm_ms_per_step_ranks',[])], 'ab', round(ab.get('exposed_comm_ms_per_step', float('nan')),2), 'p2p', [round(x,1) for x in d.get('p2p_wait_ms_per_step_ranks',[])], 'clk', d['clocks'] and d['clocks']['sm_mhz'])" || tail -3 $out.err
}
for c in 1 4 8; do run 4 gpurun_out/m2_c4_c$c.json --workload 10b --chunk $c --steps 3 --warmup 3 --no-e2e --no-ab; done
run 1 gpurun_out/m2_std_d1.json --schedule standard --steps 3 --warmup 3 --no-e2e
run 1 gpurun_out/m2_lay_d1.json --schedule layered --steps 3 --warmup 3 --no-e2e
run 4 gpurun_out/m2_std_d4.json --schedule standard --steps 3 --warmup 3 --no-e2e
