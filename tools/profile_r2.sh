# Round-2 profiles of the current build (1 x B200): plain bench, the launch list of the 1.3B step (every
# launch of 1 timed step after 3 warm-ups), then ncu --set full of the attention kernels, the GELU-backward
# GEMM and the fused LayerNorm backward.  Each ncu command runs only after the same program exited 0 plainly.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_plain.json 2> gpurun_out/r2_plain.err || exit 1
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r2_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:fwd_kernel|dkdv_kernel|dq_kernel|ln_bwd_fused" \
    -s 40 -c 8 -o gpurun_out/r2_attn python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/r2_ncu_attn.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:gemm_tc" -s 40 -c 8 -o gpurun_out/r2_gemm \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_ncu_gemm.log 2>&1
tail -2 gpurun_out/r2_ncu_attn.log gpurun_out/r2_ncu_gemm.log
