# r02aq: COO follow (pinned only) parity + timing
set -x
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_parity.py -p no:cacheprovider -k "pinned or follow or pageable or in_place or concurren or coo or COO or hyb" > gpurun_out/aq_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/aq_pytest.log
timeout 300 python scripts/e2e_formats.py 2>&1 | sed 's/^/final /'
