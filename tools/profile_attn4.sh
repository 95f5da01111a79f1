cd $GRAFT_REPO_ROOT
timeout 100 python tools/kbench.py attn > gpurun_out/kb_attn.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:fwd_kernel" -c 1 -o gpurun_out/prof_fwd_r1d python tools/kbench.py attn > gpurun_out/ncu_fwd.log 2>&1
tail -1 gpurun_out/ncu_fwd.log
