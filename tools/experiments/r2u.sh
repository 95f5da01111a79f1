cd $GRAFT_REPO_ROOT
cp paper_2106_02679_b200/liblga.so /tmp/rel.so
for rep in 1 2 3; do for v in prev cur; do
  cp exp/$v.so paper_2106_02679_b200/liblga.so
  echo "$v $(timeout 120 python tools/kbench.py ln 2>&1 | grep bwd)"
done; done
cp /tmp/rel.so paper_2106_02679_b200/liblga.so
timeout 600 python -m pytest tests/test_gpu_hbm_kernels.py -q -x -p no:cacheprovider 2>&1 | tail -1
