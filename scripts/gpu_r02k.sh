# r02k: tune graph with the bins branch forked beside the spread chain
set -x
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_tuner_corpus.py -p no:cacheprovider -k "tune or feature or corpus or predict" > gpurun_out/k_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/k_pytest.log
timeout 600 python scripts/tune_cost_probe.py > gpurun_out/k_tune_cost.txt 2>&1
head -8 gpurun_out/k_tune_cost.txt; tail -1 gpurun_out/k_tune_cost.txt
