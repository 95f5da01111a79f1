cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k attention 2>&1 | tail -1
timeout 120 python tools/kbench.py attn 2>&1 | tail -3
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"dkdv|dq_|dsum" -c 12 --csv python tools/kbench.py attn > gpurun_out/attn_bwd_ncu.csv 2>&1
python - <<'PY'
import csv,re
rows=[r for r in csv.reader(l for l in open('gpurun_out/attn_bwd_ncu.csv') if l.startswith('"'))]
h=rows[0]; ik,iv,im,iid=h.index('Kernel Name'),h.index('Metric Value'),h.index('Metric Name'),h.index('ID')
by={}
for r in rows[1:]:
    by.setdefault(int(r[iid]),{'k':re.sub(r"\(.*","",r[ik])})[r[im]]=r[iv]
for i in sorted(by): print(by[i])
PY
