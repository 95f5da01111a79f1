# the 1-GPU bench on each GPU of the box in turn (device-to-device variation under the power cap)
cd $GRAFT_REPO_ROOT
for k in 0 1 2 3; do
  CUDA_VISIBLE_DEVICES=$k python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('gpu$k', round(d['ms_per_step'],1), 'gemm', round(d['roofline']['achieved']), d['clocks'])"
done
nvidia-smi --query-gpu=index,power.limit,power.max_limit,temperature.gpu --format=csv
