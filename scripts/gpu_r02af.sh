# r02af: pinned non-DIA spmv(m, x): one-shot copy-engine path vs the host staging (SOB_PINNED_STAGED=1)
set -x
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -p no:cacheprovider -k "pinned or pageable or in_place or follow" 2>&1 | tail -2
for i in 1 2; do SOB_PINNED_STAGED=1 timeout 300 python scripts/e2e_quick.py 2>&1 | grep pinned | sed 's/^/staged /'; timeout 300 python scripts/e2e_quick.py 2>&1 | grep pinned | sed 's/^/oneshot /'; done
