# dynamic work list in the attention forward: shape check, kernel tests + kbench A/B
cd $GRAFT_REPO_ROOT
timeout 120 python tools/experiments/fwd_repro.py 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "attn or attention" -p no:cacheprovider 2>&1 | tail -1
bash tools/experiments/ab_kb.sh prev dyn
