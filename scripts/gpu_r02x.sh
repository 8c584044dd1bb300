# r02x: programmatic dependent launch through the feature / tune chain
set -x
timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_tuner_corpus.py tests/test_gpu_full_size.py tests/test_gpu_reference_suites.py -p no:cacheprovider > gpurun_out/x_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/x_pytest.log
SOB_TUNE_TRACE=1 timeout 600 python scripts/tune_cost_probe.py --ids 102,90 2>&1 | grep -E "tune\]|wall cost" | tail -7
timeout 600 python scripts/tune_cost_probe.py > gpurun_out/x_tune_cost.txt 2>&1; head -3 gpurun_out/x_tune_cost.txt | cut -c1-200; tail -1 gpurun_out/x_tune_cost.txt
