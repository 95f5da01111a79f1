# forward A/B on one box: previous build (prev) vs the working tree (new); shape check, kernel tests, trace
cd $GRAFT_REPO_ROOT
cp paper_2106_02679_b200/liblga.so exp/new.so
timeout 120 python tools/experiments/fwd_repro.py 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "attn or attention" -p no:cacheprovider 2>&1 | tail -1
for rep in 1 2 3; do for v in prev new; do
  cp exp/$v.so paper_2106_02679_b200/liblga.so
  echo "$v $(timeout 120 python tools/kbench.py attn 2>&1 | grep -E 'fwd' | sed 's/.*: //')"
done; done
cp exp/ftrace.so paper_2106_02679_b200/liblga.so
true
cp exp/new.so paper_2106_02679_b200/liblga.so
