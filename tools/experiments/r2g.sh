cd $GRAFT_REPO_ROOT
cp paper_2106_02679_b200/liblga.so /tmp/new.so
for v in notmem direct; do
  cp exp/$v.so paper_2106_02679_b200/liblga.so
  echo "== $v"; CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/experiments/fwd_repro.py 2>&1 | tail -6
done
cp /tmp/new.so paper_2106_02679_b200/liblga.so
cuobjdump -res-usage paper_2106_02679_b200/liblga.so 2>&1 | grep -A1 fwd_kernel
