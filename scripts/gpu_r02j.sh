# r02j: pageable staging with the follow-the-copy kernel (x chunks up on the copy engine as staged, y chunks out as counted)
set -x
timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_reference_suites.py -p no:cacheprovider -k "pinned or follow or pageable or in_place or spmv or concurren" > gpurun_out/j_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/j_pytest.log
timeout 900 compute-sanitizer --tool memcheck --leak-check no python scripts/sanitize_driver.py --quick > gpurun_out/j_san_memcheck.log 2>&1; echo "memcheck rc=$?"; grep -h "ERROR SUMMARY" gpurun_out/j_san_memcheck.log
for i in 1 2 3; do
  SOB_NO_FOLLOW=1 timeout 300 python scripts/e2e_quick.py 2>&1 | sed 's/^/zc /'
  timeout 300 python scripts/e2e_quick.py 2>&1 | sed 's/^/follow /'
done > gpurun_out/j_e2e.txt
for i in 1 2 3; do
  SOB_NO_FOLLOW=1 timeout 300 ./build/e2e_api 30 3 | sed 's/^/zc /'
  timeout 300 ./build/e2e_api 30 3 | sed 's/^/follow /'
done > gpurun_out/j_e2e_api.txt 2>&1
grep -E ' 2 ' gpurun_out/j_e2e.txt
cut -c1-200 gpurun_out/j_e2e_api.txt
