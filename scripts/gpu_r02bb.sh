# r02bb: pinned CSR: 8 group-range chunks into device y, each chunk's y down on copy_out as it completes, vs one FOLLOW launch storing y into mapped memory (SOB_NO_CSR_CHUNKS=1)
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "pinned or follow or concurren or in_place or csr or CSR" > gpurun_out/bb_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/bb_pytest.log; grep -E "^E |FAILED" gpurun_out/bb_pytest.log | head
for i in 1 2 3; do
  SOB_NO_CSR_CHUNKS=1 timeout 300 python scripts/e2e_formats.py 1 2>&1 | grep pinned | sed 's/^/before /'
  timeout 300 python scripts/e2e_formats.py 1 2>&1 | grep pinned | sed 's/^/after /'
done
