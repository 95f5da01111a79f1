cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k attention 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_step.py -q -x -k "bf16 or fp32_c1" 2>&1 | tail -2
timeout 120 python tools/kbench.py attn 2>&1 | tail -3
bash tools/ab.sh hints nohints
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_tc -s 60 -c 24 --csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/exp_gemm_dram.csv 2>&1
