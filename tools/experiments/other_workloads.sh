cd $GRAFT_REPO_ROOT
python bench.py --workload gpt2s --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/w_gpt2s.json 2> gpurun_out/w_gpt2s.err
tail -1 gpurun_out/w_gpt2s.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gpt2s', round(d['ms_per_step'],1), round(d['value']), 'e2e', round(d['e2e']['value']), 'gemm', round(d['roofline']['achieved']), d['kernels']['attention'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/w_gpt2s.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29655 \
  bench.py --gpus 4 --workload 10b --steps 2 --warmup 3 --no-e2e > gpurun_out/w_10b.json 2> gpurun_out/w_10b.err
tail -1 gpurun_out/w_10b.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('10b', round(d['ms_per_step'],1), round(d['value']), 'p2p', round(d['p2p_wait_ms_per_step'],1), 'gemm', round(d['roofline']['achieved']), d['comm_last_step_rank0']['p2p_send_calls'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/w_10b.err
