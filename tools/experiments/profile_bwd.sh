cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x -k attention 2>&1 | tail -2
timeout 100 python tools/kbench.py attn > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:dkdv_kernel|dq_kernel" -s 2 -c 2 -o gpurun_out/prof_bwd_r1 python tools/kbench.py attn > gpurun_out/ncu_bwd.log 2>&1
tail -1 gpurun_out/ncu_bwd.log
