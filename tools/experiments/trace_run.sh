cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -k attention 2>&1 | tail -1
timeout 60 python tools/kbench.py attn 2>&1 | grep "bwd"; timeout 60 python tools/kbench.py attn --dh 64 --heads 32 2>&1 | grep "bwd"
timeout 300 python -m pytest tests/test_gpu_step.py -q -x 2>&1 | tail -1
