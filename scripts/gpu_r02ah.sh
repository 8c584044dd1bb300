# r02ah: pinned CSR spmv(m, x) with the CSR kernels following the upload of x (y into mapped host memory)
set -x
timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_full_size.py tests/test_gpu_reference_suites.py -p no:cacheprovider -k "pinned or follow or pageable or in_place or concurren or config3 or rmat or reference" > gpurun_out/ah_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ah_pytest.log
for i in 1 2; do SOB_NO_CSR_FOLLOW=1 timeout 300 python scripts/e2e_quick.py 2>&1 | grep '^1 pinned' | sed 's/^/oneshot /'; timeout 300 python scripts/e2e_quick.py 2>&1 | grep '^1 pinned' | sed 's/^/follow /'; done
timeout 600 python scripts/ab_spmv.py after rmat,banded,hyb 2>&1 | tail -3
