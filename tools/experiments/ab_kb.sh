# kbench attention A/B of library builds (exp/<name>.so), alternated 2 rounds
cd $GRAFT_REPO_ROOT
cp paper_2106_02679_b200/liblga.so /tmp/rel.so
for rep in 1 2; do for v in "$@"; do
  cp exp/$v.so paper_2106_02679_b200/liblga.so
  echo "$v $(timeout 120 python tools/kbench.py attn 2>&1 | grep -E 'fwd|bwd 5-mm  ' | sed 's/.*: //' | cut -c1-24 | tr '\n' ' ')"
done; done
cp /tmp/rel.so paper_2106_02679_b200/liblga.so
