cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "attn or attention" -p no:cacheprovider 2>&1 | tail -1
cp paper_2106_02679_b200/liblga.so /tmp/rel.so
for rep in 1 2; do for v in prev g4; do
  cp exp/$v.so paper_2106_02679_b200/liblga.so
  echo "$v C2 $(timeout 120 python tools/kbench.py attn --dh 64 --seq 1024 --nseq 32 --heads 12 2>&1 | grep 'bwd 5-mm  ' | sed 's/.*: //')"
done; done
cp /tmp/rel.so paper_2106_02679_b200/liblga.so
