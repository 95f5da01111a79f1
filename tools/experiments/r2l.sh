# attention-forward trace with the item-boundary events (exp/ftrace.so)
cd $GRAFT_REPO_ROOT
cp paper_2106_02679_b200/liblga.so /tmp/rel.so
cp exp/ftrace.so paper_2106_02679_b200/liblga.so
timeout 120 python tools/fwd_trace.py 2>&1 | tail -62
cp /tmp/rel.so paper_2106_02679_b200/liblga.so
