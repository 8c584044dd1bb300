# r02as: csr_long_pieces / csr_long_fixup with PDL (each waits at entry) vs plain launches
for i in 1 2 3; do
  SOB_NO_PDL_FIXUP=1 timeout 600 python scripts/ab_spmv.py plain rmat,lap 2>&1 | tail -2
  timeout 600 python scripts/ab_spmv.py pdl rmat,lap 2>&1 | tail -2
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_size.py -m gpu -q -x -p no:cacheprovider -k "csr or CSR or hdc or HDC or long or rmat or coo" 2>&1 | tail -2
