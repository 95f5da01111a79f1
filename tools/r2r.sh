cd $GRAFT_REPO_ROOT
cp paper_2106_02679_b200/liblga.so /tmp/rel.so
cp exp/dtrace.so paper_2106_02679_b200/liblga.so
timeout 120 python tools/dkv_trace.py 2>&1 | tail -80
cp /tmp/rel.so paper_2106_02679_b200/liblga.so
