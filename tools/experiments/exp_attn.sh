# A/B of attention-forward builds (exp/<v>.so): kbench forward/backward timing, alternated, 3 rounds
cd $GRAFT_REPO_ROOT
cp paper_2106_02679_b200/liblga.so /tmp/rel.so
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k attention 2>&1 | tail -1
for rep in 1 2 3; do for v in "$@"; do
  cp exp/$v.so paper_2106_02679_b200/liblga.so
  echo "$v $(timeout 120 python tools/kbench.py attn 2>&1 | grep -E 'fwd|bwd' | sed 's/.*: //' | cut -c1-30 | tr '\n' ' ')"
done; done
cp /tmp/rel.so paper_2106_02679_b200/liblga.so
