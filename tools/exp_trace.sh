cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x -k attention 2>&1 | tail -2
timeout 60 python tools/kbench.py attn > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:fwd_kernel" -s 3 -c 1 -o gpurun_out/prof_fwd_r1e python tools/kbench.py attn > gpurun_out/ncu_fwd.log 2>&1
tail -1 gpurun_out/ncu_fwd.log
