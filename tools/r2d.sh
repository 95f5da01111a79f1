# Round-2: the multi-rank resume test (load_state now collective) x3, the full GPU suite (no -x), then the
# attention-forward pipeline trace (LGA_FWD_TRACE build in exp/ftrace.so).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_dist.py -q -k checkpoint -p no:cacheprovider 2>&1 | tail -1; done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2d_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2d_pytest.log
tail -3 gpurun_out/r2d_pytest.log
cp paper_2106_02679_b200/liblga.so /tmp/rel.so
cp exp/ftrace.so paper_2106_02679_b200/liblga.so
timeout 120 python tools/fwd_trace.py > gpurun_out/r2d_fwd_trace.txt 2>&1
cp /tmp/rel.so paper_2106_02679_b200/liblga.so
cat gpurun_out/r2d_fwd_trace.txt
