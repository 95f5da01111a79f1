# attention backward A/B: previous build (prev) vs working tree (cur), kbench backward; kernel tests
cd $GRAFT_REPO_ROOT
true
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "attn or attention" -p no:cacheprovider 2>&1 | tail -1
for rep in 1 2; do for v in prev cur; do
  cp exp/$v.so paper_2106_02679_b200/liblga.so
  echo "== $v"; timeout 120 python tools/kbench.py attn 2>&1 | grep bwd
done; done
cp exp/cur.so paper_2106_02679_b200/liblga.so
