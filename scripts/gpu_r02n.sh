# r02n: tune plan times both CSR sweeps once and keeps the faster
set -x
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_tuner_corpus.py -p no:cacheprovider -k "tune or feature or corpus or predict or concurren" > gpurun_out/n_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/n_pytest.log
timeout 600 python scripts/tune_cost_probe.py > gpurun_out/n_tune_cost.txt 2>&1
head -6 gpurun_out/n_tune_cost.txt | cut -c1-220; tail -1 gpurun_out/n_tune_cost.txt
