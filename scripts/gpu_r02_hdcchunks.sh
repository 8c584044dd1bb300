# Pinned HDC (both parts) chunk pipeline (1 GPU): the follow / pinned parity tests, then the
# HYB-shaped matrix's HDC pinned wall time with the chunk pipelines on and off
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "coo or pinned or follow or hdc or host" > gpurun_out/hc_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/hc_pytest.log
timeout 300 python scripts/e2e_formats.py 1,5 > gpurun_out/hc_e2e_formats.txt 2>&1
SOB_NO_CSR_CHUNKS=1 timeout 300 python scripts/e2e_formats.py 1,5 > gpurun_out/hc_e2e_formats_off.txt 2>&1
cat gpurun_out/hc_e2e_formats.txt; echo "--- SOB_NO_CSR_CHUNKS=1"; cat gpurun_out/hc_e2e_formats_off.txt
