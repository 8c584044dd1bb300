# r02am: pageable spmv(m, x) on CSR / ELL with staged x chunks uploaded behind the FOLLOW kernels
set -x
timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_reference_suites.py -p no:cacheprovider -k "pinned or follow or pageable or in_place or concurren or spmv or reference" > gpurun_out/am_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/am_pytest.log
for i in 1 2; do SOB_NO_CSR_FOLLOW=1 timeout 300 python scripts/e2e_quick.py 2>&1 | grep -E 'pageable' | sed 's/^/staged /'; timeout 300 python scripts/e2e_quick.py 2>&1 | grep -E 'pageable' | sed 's/^/follow /'; done
