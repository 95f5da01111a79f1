# Config 4 (~10B: L=48, d=4096, s=2048, N=32) with the modular pipeline.  On a 4-GPU box: P=4 x D=1.
cd $GRAFT_REPO_ROOT
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29644 \
  bench.py --gpus 4 --workload 10b --steps 2 --warmup 3 --no-e2e 2> gpurun_out/b10.err | tail -1 > gpurun_out/b10.json
tail -3 gpurun_out/b10.err
python -c "import json; d=json.load(open('gpurun_out/b10.json')); print(d['ms_per_step'], d['value'], d['p2p_wait_ms_per_step'], d['exposed_comm_ms_per_step'], d['comm_last_step_rank0'], d['roofline']['achieved'])"
