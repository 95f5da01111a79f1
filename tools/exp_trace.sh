cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x -k "epilogue or tc_gemm" 2>&1 | tail -2
timeout 300 python -m pytest tests/test_gpu_step.py -q -x 2>&1 | tail -2
timeout 100 python tools/kbench.py gemm 2>&1 | tail -9
python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_tc2_kernel -s 200 -c 6 python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e 2>&1 | grep -E "gemm_tc2|duration|hmma" | head -18
