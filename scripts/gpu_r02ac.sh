# r02ac: pinned spmv(m, x) with kernels storing y into mapped host memory (CSR/ELL/COO...) vs the staged path
set -x
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -p no:cacheprovider -k "pinned or follow or pageable or in_place or concurren or store_y" > gpurun_out/ac_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ac_pytest.log
for i in 1 2; do SOB_NO_MAPPED_Y=1 timeout 300 python scripts/e2e_quick.py 2>&1 | grep pinned | sed 's/^/staged /'; timeout 300 python scripts/e2e_quick.py 2>&1 | grep pinned | sed 's/^/mapped /'; done
