# SURVEY 8(f) variants, measured: C3 on 4 GPUs (default / keep params / unpartitioned / no recompute) and
# C4 (10B, P=4) modular vs contiguous pipeline.  One JSON line per run in gpurun_out/var_<name>.json.
cd $GRAFT_REPO_ROOT
run4() {  # name, extra args
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) \
    bench.py --gpus 4 --steps 3 --warmup 3 --no-e2e $2 > gpurun_out/var_$1.json 2> gpurun_out/var_$1.err
  tail -1 gpurun_out/var_$1.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['comm_last_step_rank0']
print('$1', round(d['ms_per_step'],1), round(d['value']), 'exposed', round(d['exposed_comm_ms_per_step'],2), 'p2p', round(d['p2p_wait_ms_per_step'],1),
      'ag', c['ag_calls'], c['ag_bytes'], 'rs', c['rs_calls'], c['rs_bytes'], 'ar', c['allreduce_calls'], c.get('allreduce_bytes'), 'recomp', c['recompute_units'], 'p2p', c['p2p_send_calls'], d['clocks']['sm_mhz'])" \
    || tail -4 gpurun_out/var_$1.err
}
run4 c3_default ""
run4 c3_keep "--keep-params"
run4 c3_unpart "--unpartitioned"
run4 c3_norecomp "--no-recompute"
run4 c4_modular "--workload 10b"
run4 c4_contiguous "--workload 10b --pipeline contiguous"
