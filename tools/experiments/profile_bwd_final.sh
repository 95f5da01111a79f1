# ncu --set full of the backward kernels (dK/dV, dQ, fused LayerNorm backward) inside the 1.3B step
cd $GRAFT_REPO_ROOT
python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:dkdv_kernel|dq_kernel|ln_bwd_fused" -c 6 \
    -o gpurun_out/final_bwd python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bwd2.log 2>&1
echo done
