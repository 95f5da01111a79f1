cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x -k attention 2>&1 | tail -2
echo "== release (3)"; timeout 60 python tools/kbench.py attn 2>&1 | grep bwd
cp paper_2106_02679_b200/liblga.so /tmp/rel.so
for f in exp/*.so; do cp $f paper_2106_02679_b200/liblga.so; echo "== $f"; timeout 60 python tools/kbench.py attn 2>&1 | grep bwd; done
cp /tmp/rel.so paper_2106_02679_b200/liblga.so
