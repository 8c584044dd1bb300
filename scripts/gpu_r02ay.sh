# r02ay: pinned follow calls queue the upload first and wait for their kernels (event), not for the sentinel refill
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "pinned or follow or pageable or concurren or coo or in_place" > gpurun_out/ay_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ay_pytest.log
for i in 1 2 3; do
  SOB_FOLLOW_KERNEL_FIRST=1 timeout 300 python scripts/e2e_quick.py 2>&1 | grep pinned | sed 's/^/before /'
  timeout 300 python scripts/e2e_quick.py 2>&1 | grep pinned | sed 's/^/after /'
done
