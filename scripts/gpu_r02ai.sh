# r02ai: sanitizers over the driver incl. the pinned DIA / CSR follow kernels
set -x
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t $( [ $t = memcheck ] && echo --leak-check no ) python scripts/sanitize_driver.py > gpurun_out/ai_sanitizer_$t.log 2>&1; echo "$t rc=$?"; grep -h "ERROR SUMMARY\|RACECHECK SUMMARY\|driver done" gpurun_out/ai_sanitizer_$t.log | tail -2
done
