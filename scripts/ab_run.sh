set -x
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_full_size.py -k "hyb or HYB or rmat or random or switch or pageable" 2>&1 | tail -3
for i in 1 2; do
SOB_HYB_SERIAL=1 timeout 300 python scripts/ab_spmv.py serial rmat,unif,hyb
timeout 300 python scripts/ab_spmv.py fork rmat,unif,hyb
done
