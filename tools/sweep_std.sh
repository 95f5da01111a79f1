# STANDARD (with all-gather prefetch) vs LAYERED at D=4, selected N; appends to gpurun_out/sweep_std.jsonl
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/sweep_std.jsonl
: > $OUT
for cfg in "standard 1" "standard 4" "standard 16" "layered 16"; do
  set -- $cfg
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29644 \
    bench.py --gpus 4 --steps 2 --warmup 3 --n-micro $2 --schedule $1 --no-e2e 2>/dev/null | tail -1 >> $OUT
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
          f"exposed_comm_ms={d['exposed_comm_ms_per_step']:7.2f} ag_bytes={k['ag_bytes']:14d} rs_bytes={k['rs_bytes']:14d}")
PY
