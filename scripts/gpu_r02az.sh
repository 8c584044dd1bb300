# r02az: pageable COO / HYB: follow kernels into device y, y down chunk by chunk (event each) vs the staged path (SOB_PAGEABLE_COO_STAGED=1)
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "pinned or follow or pageable or concurren or coo or in_place" > gpurun_out/az_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/az_pytest.log; grep -E "^E |FAILED" gpurun_out/az_pytest.log | head
for i in 1 2 3; do
  SOB_PAGEABLE_COO_STAGED=1 timeout 300 python scripts/e2e_formats.py 0,4 2>&1 | grep pageable | sed 's/^/staged /'
  timeout 300 python scripts/e2e_formats.py 0,4 2>&1 | grep pageable | sed 's/^/follow /'
done
