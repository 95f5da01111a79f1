cd $GRAFT_REPO_ROOT
N=${1:-4}
for n in 1 2 4 8; do
  if [ $n -gt $N ]; then break; fi
  if [ $n -eq 1 ]; then
    timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/scale_$n.json 2> gpurun_out/scale_$n.err
  else
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2950$n bench.py --gpus $n --steps 4 --warmup 3 --no-e2e > gpurun_out/scale_$n.json 2> gpurun_out/scale_$n.err
  fi
  tail -1 gpurun_out/scale_$n.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($n, round(d['ms_per_step'],1), round(d['value']), 'exposed', round(d['exposed_comm_ms_per_step'],2), 'gemm', round(d['roofline']['achieved']), d['comm_last_step_rank0']['ag_bytes'], d['clocks'])" || tail -5 gpurun_out/scale_$n.err
done
