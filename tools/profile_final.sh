# Round profiles of the current build (1 x B200): plain bench, launch list of one 1.3B step, ncu --set full
# of the top kernels.  Each ncu command runs only after the same program exited 0 without ncu.
cd $GRAFT_REPO_ROOT
python bench.py --steps 5 --warmup 3 > gpurun_out/final_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -s 1900 -c 1100 --csv --log-file gpurun_out/launches_final.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_tc2_kernel -s 200 -c 6 -o gpurun_out/final_gemm \
    python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:fwd_kernel|dkdv_kernel|dq_kernel|ln_bwd_fused" -s 12 -c 8 \
    -o gpurun_out/final_attn python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ncu_attn.log 2>&1
tail -2 gpurun_out/ncu_gemm.log gpurun_out/ncu_attn.log
