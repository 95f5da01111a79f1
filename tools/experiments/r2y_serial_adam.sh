# A/B at D = 4 (C3): RS + AdamW overlapped on the comm stream (default) vs serialized with the compute stream
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() {   # out env...
  local out=$1; shift
  env "$@" timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-ab > $out 2> $out.err
  tail -1 $out | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$out', round(d['ms_per_step'],1), round(d['value']), 'stall', [round(x,2) for x in d['exposed_comm_ms_per_step_ranks']], 'clk', d['clocks']['sm_mhz'])" || tail -3 $out.err
}
for rep in 1 2; do
  run gpurun_out/sa_overlap_$rep.json LGA_NOTHING=1
  run gpurun_out/sa_serial_$rep.json LGA_EXP_SERIAL_ADAM=1
done
