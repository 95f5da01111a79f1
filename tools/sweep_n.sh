# Config 5: micro-batch-count sweep at the 1.3B shape, layered vs standard accumulation,
# D GPUs; one bench line per (schedule, N) -> gpurun_out/sweep_D<d>.jsonl
cd $GRAFT_REPO_ROOT
D=${1:-2}
OUT=gpurun_out/sweep_D$D.jsonl
: > $OUT
for sched in layered standard; do
  for N in 1 2 4 8 16 32; do
    if [ "$sched" = "standard" ] && [ $N -gt 16 ]; then continue; fi
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $D --master-addr 127.0.0.1 --master-port 2961$D \
      bench.py --gpus $D --steps 2 --warmup 3 --n-micro $N --schedule $sched --no-e2e 2>/dev/null | tail -1 >> $OUT
  done
done
python - "$OUT" <<'PY'
import json, sys
for line in open(sys.argv[1]):
    try:
        d = json.loads(line)
    except Exception:
        continue
    c = d["config"]; k = d["comm_last_step_rank0"]
    print(f"{c['schedule']:9s} N={c['n_micro']:3d} D={c['dp']} ms/step={d['ms_per_step']:8.1f} tok/s={d['value']:10.0f} "
          f"exposed_comm_ms={d['exposed_comm_ms_per_step']:7.2f} ag_calls={k['ag_calls']:5d} ag_bytes={k['ag_bytes']:14d} "
          f"rs_calls={k['rs_calls']:5d} rs_bytes={k['rs_bytes']:14d}")
PY
