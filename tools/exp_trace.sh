cd $GRAFT_REPO_ROOT
cp paper_2106_02679_b200/liblga.so /tmp/rel.so
echo "== release"; timeout 120 python tools/kbench.py attn 2>&1 | grep bwd
for f in exp/*.so; do cp $f paper_2106_02679_b200/liblga.so; echo "== $f"; timeout 120 python tools/kbench.py attn 2>&1 | grep bwd;
  case $f in *TRACE*) timeout 120 python tools/bwd_trace.py 0 > gpurun_out/bwd_trace_$(basename $f .so).txt 2>&1;; esac; done
cp /tmp/rel.so paper_2106_02679_b200/liblga.so
