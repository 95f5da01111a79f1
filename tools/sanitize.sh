# compute-sanitizer over the LGA step (tools/sanitize_step.py); logs -> gpurun_out/sanitize_<tool>.log
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/sanitize_step.py all > gpurun_out/sanitize_plain.log 2>&1 || { tail -5 gpurun_out/sanitize_plain.log; exit 1; }
for tool in memcheck synccheck racecheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 python tools/sanitize_step.py all \
      > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Invalid|Race|Barrier" gpurun_out/sanitize_$tool.log | head -5
done
