cd $GRAFT_REPO_ROOT
for cfg in "1 256 2 128" "1 2048 1 128" "1 2048 16 128" "2 2048 16 128" "16 512 16 128" "4 2048 16 128" "16 2048 16 128"; do
  timeout 30 python tools/attn_sizes.py $cfg 2>&1 | tail -1
done
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x -k attention 2>&1 | tail -2
timeout 60 python tools/kbench.py attn 2>&1 | grep -v "^$"; timeout 60 python tools/kbench.py attn --dh 64 --heads 32 2>&1 | grep "bwd\|tcgen"
