# r02ag: spread walk with a sequential head (SOB_WALK_HEAD rows; 0 = the record walk from row 0)
set -x
timeout 1500 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_tuner_corpus.py tests/test_gpu_full_size.py -p no:cacheprovider -k "feature or spread or corpus or config or random or tune or arrow" > gpurun_out/ag_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ag_pytest.log
SOB_WALK_HEAD=0 timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -p no:cacheprovider -k "spread or feature" 2>&1 | tail -1
for hd in 0 512 1024 2048; do SOB_WALK_HEAD=$hd timeout 600 python scripts/tune_cost_probe.py 2>&1 | tail -1 | sed "s/^/head$hd /"; done
for hd in 0 1024; do SOB_WALK_HEAD=$hd timeout 600 python scripts/tune_cost_probe.py --ids 102,90,30,474 2>&1 | grep '^{' | cut -c1-160 | sed "s/^/head$hd /"; done
