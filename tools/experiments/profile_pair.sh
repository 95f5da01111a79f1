cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "tc_gemm" 2>&1 | tail -3
echo "--- pair (default)"; timeout 100 python tools/kbench.py gemm 2>&1 | tail -9
echo "--- single-CTA"; LGA_GEMM_PAIR=0 timeout 100 python tools/kbench.py gemm 2>&1 | tail -9
timeout 300 python -m pytest tests/test_gpu_step.py -q -x 2>&1 | tail -2
for v in 1 0; do LGA_GEMM_PAIR=$v timeout 100 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pair=$v', d['ms_per_step'], d['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'])"; done
timeout 100 python tools/kbench.py attn > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k "regex:dkdv_kernel|dq_kernel|dsum" -c 6 --csv python tools/kbench.py attn 2>/dev/null | grep -E "dkdv|dq_kernel|dsum" | awk -F'","' '{print $5, $13, $15}' | cut -c1-150
