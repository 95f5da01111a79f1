# refresh the committed launch list on the final build (1 x B200); ncu only after the plain run exited 0
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -k 10 200 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/lr_plain.json 2> gpurun_out/lr_plain.err || { tail -5 gpurun_out/lr_plain.err; exit 1; }
tail -1 gpurun_out/lr_plain.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('plain', round(d['ms_per_step'],1), d['gpu_launches'], d['roofline'])"
timeout -k 10 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 1900 -c 1100 --csv --log-file gpurun_out/launches_r1_final.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/lr_ncu.log 2>&1
echo "ncu rc=$?"; wc -l gpurun_out/launches_r1_final.csv
