cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -k attention 2>&1 | grep -E "FAILED|passed|failed|assert|Error" | head -20
timeout 60 python tools/kbench.py attn 2>&1 | grep "fwd tc"
