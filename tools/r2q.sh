# ncu --set full of the current build's top kernels in the C3 step (after the plain run exits 0)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k "regex:gemm_tc2_kernel" -s 200 -c 6 -o gpurun_out/r2q_gemm \
    python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r2q_ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:fwd_kernel|dkdv_kernel|dq_from_ds" -s 12 -c 6 \
    -o gpurun_out/r2q_attn python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r2q_ncu_attn.log 2>&1
python tools/ncu_summary.py gpurun_out/r2q_gemm.ncu-rep
python tools/ncu_summary.py gpurun_out/r2q_attn.ncu-rep
