# Round-2 multi-GPU measurements on one 4-GPU box (all through bench.py, peer-memory data path):
#  1. weak scaling at C3: N = 1, 2, 4 (N > 1 with the no-comm A/B)       -> gpurun_out/m_scale_<n>.json
#  2. config 5 sweep at C3, D = 2 and 4: LAYERED N = 1..64, STANDARD N = 1..16 -> gpurun_out/m_sweep_D<d>.jsonl
#  3. C4 (10B) modular pipeline P = 4 x D = 1, chunk 1 and 2               -> gpurun_out/m_c4_c<c>.json
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
  tail -1 $out | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; ab=d.get('exposed_comm_ab') or {}; print('$out', c['schedule'], 'N', c['n_micro'], 'dp', c['dp'], 'pp', c['pp'], 'ms', round(d['ms_per_step'],1), 'tok/s', round(d['value']), 'stall', round(d['exposed_comm_ms_per_step'],2), 'ab', round(ab.get('exposed_comm_ms_per_step', float('nan')),2), 'p2p', round(d['p2p_wait_ms_per_step'],2), 'clk', d['clocks'] and d['clocks']['sm_mhz'])" || tail -3 $out.err
}
for n in 1 2 4; do run $n gpurun_out/m_scale_$n.json --steps 10 --warmup 3 --no-e2e; done
for D in 2 4; do
  : > gpurun_out/m_sweep_D$D.jsonl
  for sched in layered standard; do
    for N in 1 4 16 64; do
      if [ "$sched" = "standard" ] && [ $N -gt 16 ]; then continue; fi
      run $D gpurun_out/m_sw_${sched}_${N}_$D.json --steps 3 --warmup 3 --n-micro $N --schedule $sched --no-e2e --no-ab
      tail -1 gpurun_out/m_sw_${sched}_${N}_$D.json >> gpurun_out/m_sweep_D$D.jsonl
    done
  done
done
for c in 1 2; do run 4 gpurun_out/m_c4_c$c.json --workload 10b --chunk $c --steps 3 --warmup 3 --no-e2e --no-ab; done
