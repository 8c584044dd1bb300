# Pinned COO chunk pipeline (1 GPU): the COO / follow parity tests, then config 2 COO
# pinned wall time with the chunk pipeline on and off, and its difference to the device multiply
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "coo or pinned or follow" > gpurun_out/cc_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/cc_pytest.log
for k in 1 2; do
  timeout 300 python scripts/coo_chunk_check.py
  SOB_NO_COO_CHUNKS=1 timeout 300 python scripts/coo_chunk_check.py
done 2>&1 | tee gpurun_out/cc_check.txt
timeout 300 python scripts/e2e_formats.py 0 > gpurun_out/cc_e2e_formats.txt 2>&1; cat gpurun_out/cc_e2e_formats.txt
