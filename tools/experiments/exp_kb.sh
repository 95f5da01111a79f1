# A/B of builds (exp/<v>.so) on one kbench section: bash tools/experiments/exp_kb.sh <attn|gemm|ln> v1 v2 ...
cd $GRAFT_REPO_ROOT
what=$1; shift
cp paper_2106_02679_b200/liblga.so /tmp/rel.so
for rep in 1 2 3; do for v in "$@"; do
  cp exp/$v.so paper_2106_02679_b200/liblga.so
  echo "$v | $(timeout 120 python tools/kbench.py $what 2>&1 | sed 's/.*: //' | cut -c1-32 | tr '\n' '|')"
done; done
cp /tmp/rel.so paper_2106_02679_b200/liblga.so
