cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x -k attention 2>&1 | tail -2
timeout 120 python tools/kbench.py attn 2>&1 | grep -v "^$"; timeout 120 python tools/kbench.py attn --dh 64 --heads 32 2>&1 | grep "bwd\|tcgen"
cp paper_2106_02679_b200/liblga.so /tmp/rel.so
cp exp/fwdtrace.so paper_2106_02679_b200/liblga.so
timeout 120 python tools/fwd_trace.py > gpurun_out/fwd_trace.txt 2>&1
cp /tmp/rel.so paper_2106_02679_b200/liblga.so
