cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" 2>&1 | tail -2
bash tools/ab.sh hints gm
cp exp/gm.so paper_2106_02679_b200/liblga.so
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_tc -s 60 -c 40 --csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/exp_gemm_dram_gm.csv 2>&1
