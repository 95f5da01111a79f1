cd $GRAFT_REPO_ROOT
timeout 100 python tools/kbench.py attn > gpurun_out/kb_attn.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:dkdv_kernel|dq_kernel|fwd_kernel" -c 6 -o gpurun_out/prof_attn_r1c python tools/kbench.py attn > gpurun_out/ncu_attn3.log 2>&1
tail -2 gpurun_out/ncu_attn3.log
