# dK/dV drain with early accumulator release: kernel tests, kbench A/B (prev vs cur), trace
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "attn or attention" -p no:cacheprovider 2>&1 | tail -1
bash tools/experiments/ab_kb.sh prev cur
bash tools/r2r.sh | tail -12
