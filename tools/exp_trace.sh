cd $GRAFT_REPO_ROOT
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:ln_bwd -c 4 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep -E "ln_bwd|duration|bytes" | head -16
