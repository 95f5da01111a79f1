# time kbench attn with each exp/*.so swapped in (timing-only experiment builds)
cd $GRAFT_REPO_ROOT
cp paper_2106_02679_b200/liblga.so /tmp/rel.so
echo "== release"; timeout 120 python tools/kbench.py attn 2>&1 | grep bwd
for f in exp/*.so; do cp $f paper_2106_02679_b200/liblga.so; echo "== $f"; timeout 120 python tools/kbench.py attn 2>&1 | grep bwd; done
cp /tmp/rel.so paper_2106_02679_b200/liblga.so
