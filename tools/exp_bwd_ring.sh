# ring-depth experiment for the attention backward (exp/*.so built with LGA_EXTRA_DEFINES)
cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x -k attn 2>&1 | tail -2
timeout 300 python -m pytest tests/test_gpu_step.py -q -x 2>&1 | tail -2
echo "== release"; timeout 120 python tools/kbench.py attn 2>&1 | grep bwd; timeout 120 python tools/kbench.py attn --dh 64 --heads 32 2>&1 | grep bwd
cp paper_2106_02679_b200/liblga.so /tmp/rel.so
cp exp/nst2.so paper_2106_02679_b200/liblga.so; echo "== dkv NST=2 (dh128)"; timeout 120 python tools/kbench.py attn 2>&1 | grep bwd
cp exp/deep64.so paper_2106_02679_b200/liblga.so; echo "== dh64 NST 6/8"; timeout 120 python tools/kbench.py attn --dh 64 --heads 32 2>&1 | grep bwd
cp /tmp/rel.so paper_2106_02679_b200/liblga.so
