set -x
cd $GRAFT_REPO_ROOT
python tools/kbench.py attn gemm > gpurun_out/kb_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:fwd_kernel|dkdv_kernel|dq_kernel|gemm_tc_kernel" -s 3 -c 12 -o gpurun_out/prof_attn_r1 python tools/kbench.py attn gemm > gpurun_out/ncu_attn.log 2>&1
tail -3 gpurun_out/ncu_attn.log
