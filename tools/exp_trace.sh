cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" 2>&1 | tail -2
timeout 300 python -m pytest tests/test_gpu_step.py -q -x 2>&1 | tail -2
timeout 100 python tools/kbench.py gemm 2>&1 | tail -3
bash tools/ab.sh old new
