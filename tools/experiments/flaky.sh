# repeat the multi-GPU and step suites to catch rare races (flags, graph replay, peer-memory DP)
cd $GRAFT_REPO_ROOT
for rep in 1 2 3; do
  echo "== rep $rep"
  timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_step.py -q -p no:randomly 2>&1 | tail -1
done
