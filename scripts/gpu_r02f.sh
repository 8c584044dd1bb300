# r02f: cp.async-staged CSR gathers (csr_async_kernel) vs the register-staged kernel (SOB_CSR_SYNC=1)
set -x
timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_full_size.py -p no:cacheprovider > gpurun_out/f_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/f_pytest.log
for i in 1 2; do
SOB_CSR_SYNC=1 timeout 600 python scripts/ab_spmv.py sync rmat,unif,hyb,banded,lap
timeout 600 python scripts/ab_spmv.py async rmat,unif,hyb,banded,lap
done > gpurun_out/f_ab.txt 2>&1
cat gpurun_out/f_ab.txt
