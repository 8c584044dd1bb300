# r02y: sweep mode 2 (all-direct global atomics) -- parity with the mode forced, and the tune plan's 3-way choice
set -x
SOB_FEAT_ENTRY=2 timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_tuner_corpus.py tests/test_gpu_full_size.py -p no:cacheprovider -k "feature or corpus or rmat or random or config" > gpurun_out/y_pytest_forced2.log 2>&1; echo "pytest forced2 rc=$?"; tail -2 gpurun_out/y_pytest_forced2.log
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_tuner_corpus.py -p no:cacheprovider -k "tune or feature or corpus" > gpurun_out/y_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/y_pytest.log
for e in 0 1 2; do SOB_FEAT_ENTRY=$e timeout 600 python scripts/tune_rmat_probe.py 2>&1 | sed "s/^/mode$e /"; done
timeout 600 python scripts/tune_rmat_probe.py 2>&1 | sed "s/^/auto /"
timeout 600 python scripts/tune_cost_probe.py > gpurun_out/y_tune_cost.txt 2>&1; tail -1 gpurun_out/y_tune_cost.txt
