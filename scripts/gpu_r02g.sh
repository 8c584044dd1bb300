# r02g: follow-the-copy pinned spmv (dia_follow_kernel): parity, sanitizers, e2e A/B vs zero-copy
set -x
timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -p no:cacheprovider -k "pinned or follow or pageable or in_place" > gpurun_out/g_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/g_pytest.log
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t $( [ $t = memcheck ] && echo --leak-check no ) python scripts/sanitize_driver.py --quick > gpurun_out/g_san_$t.log 2>&1; echo "$t rc=$?"; grep -h "ERROR SUMMARY\|RACECHECK SUMMARY\|done" gpurun_out/g_san_$t.log | tail -2
done
for i in 1 2 3; do
  SOB_NO_FOLLOW=1 timeout 300 python scripts/e2e_quick.py 2>&1 | sed 's/^/zc /'
  timeout 300 python scripts/e2e_quick.py 2>&1 | sed 's/^/follow /'
done > gpurun_out/g_e2e.txt
cat gpurun_out/g_e2e.txt | cut -c1-300
