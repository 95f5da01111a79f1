# attention-forward trace: per-tile pipeline and per-item spans of CTA 0, CTA end spread (exp/ftrace.so)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python tools/kbench.py attn 2>&1 | tail -4
cp paper_2106_02679_b200/liblga.so /tmp/rel.so
cp exp/ftrace.so paper_2106_02679_b200/liblga.so
timeout 120 python tools/fwd_trace.py > gpurun_out/r2e_fwd_trace.txt 2>&1
cp /tmp/rel.so paper_2106_02679_b200/liblga.so
cat gpurun_out/r2e_fwd_trace.txt
