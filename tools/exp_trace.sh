cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x -k attention 2>&1 | tail -2
timeout 60 python tools/kbench.py attn 2>&1 | grep -v "^$"; timeout 60 python tools/kbench.py attn --dh 64 --heads 32 2>&1 | grep "bwd\|tcgen"
timeout 300 python -m pytest tests/test_gpu_step.py -q -x 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"dq_kernel|dkdv_kernel" -c 4 python tools/kbench.py attn 2>&1 | grep -E "dq_k|dkdv_k|duration" | head -8
