set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "random_conversions or rmat or even_row or hdc_with or config1 or banded" 2>&1 | tail -3
for i in 1 2; do
AB_ROOT=build/ab_old timeout 300 python scripts/ab_spmv.py old rmat,unif,hyb,lap,banded
AB_ROOT=build/ab_a timeout 300 python scripts/ab_spmv.py A rmat,unif,hyb,lap,banded
timeout 300 python scripts/ab_spmv.py B rmat,unif,hyb,lap,banded
done
