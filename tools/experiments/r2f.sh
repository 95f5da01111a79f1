# attention forward with dedicated epilogue warps: shape check, kernel tests, kbench A/B against the previous build, trace
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out exp
cp paper_2106_02679_b200/liblga.so exp/new.so
timeout 120 python tools/experiments/fwd_repro.py 2>&1 | tail -6
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "attn or attention" -p no:cacheprovider 2>&1 | tail -2
for rep in 1 2 3; do for v in base new; do
  cp exp/$v.so paper_2106_02679_b200/liblga.so
  echo "$v $(timeout 120 python tools/kbench.py attn 2>&1 | grep -E 'fwd' | sed 's/.*: //')"
done; done
cp exp/ftrace.so paper_2106_02679_b200/liblga.so
timeout 120 python tools/fwd_trace.py > gpurun_out/r2f_fwd_trace.txt 2>&1
cp exp/new.so paper_2106_02679_b200/liblga.so
tail -40 gpurun_out/r2f_fwd_trace.txt
