cd $GRAFT_REPO_ROOT
timeout 30 python tools/attn_debug.py 128:200 64:200 128:2048 > /dev/null && timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k attention 2>&1 | tail -2
timeout 100 python tools/kbench.py attn > gpurun_out/kb_attn.log 2>&1 && cat gpurun_out/kb_attn.log && \
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k "regex:fat|dsum" -c 8 --csv python tools/kbench.py attn 2>/dev/null | grep -E "fwd_kernel|dkdv|dq_kernel|dsum" | cut -c1-250
