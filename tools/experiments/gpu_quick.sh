# quick GPU check: attention kernel tests, single-GPU step parity, attention kbench (+ exp/*.so variants)
cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x -k attention 2>&1 | tail -2
timeout 300 python -m pytest tests/test_gpu_step.py -q -x 2>&1 | tail -2
timeout 120 python tools/kbench.py attn 2>&1 | grep -v "^$"; timeout 120 python tools/kbench.py attn --dh 64 --heads 32 2>&1 | grep "bwd\|tcgen"
cp paper_2106_02679_b200/liblga.so /tmp/rel.so
for f in exp/*.so; do [ -e "$f" ] || continue; cp $f paper_2106_02679_b200/liblga.so; echo "== $f"; timeout 120 python tools/kbench.py attn 2>&1 | grep bwd;
  case $f in *TRACE*) timeout 120 python tools/bwd_trace.py 0 > gpurun_out/bwd_trace_$(basename $f .so).txt 2>&1;; esac; done
cp /tmp/rel.so paper_2106_02679_b200/liblga.so
