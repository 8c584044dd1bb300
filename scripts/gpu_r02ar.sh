# r02ar: fix-up kernels (coo_fixup, csr_long_pieces/fixup) launched with PDL vs plain launches (SOB_NO_PDL_FIXUP=1)
set -x
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/ar_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ar_pytest.log
for i in 1 2 3; do
  SOB_NO_PDL_FIXUP=1 timeout 600 python scripts/ab_spmv.py plain lap,banded,rmat,hyb 2>&1 | tail -4
  timeout 600 python scripts/ab_spmv.py pdl lap,banded,rmat,hyb 2>&1 | tail -4
done
for i in 1 2; do
  SOB_NO_PDL_FIXUP=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-config4 --no-config5 --no-cpu-baseline > gpurun_out/ar_bench_plain_$i.json 2>/dev/null
  timeout 600 python bench.py --steps 20 --warmup 5 --no-config4 --no-config5 --no-cpu-baseline > gpurun_out/ar_bench_pdl_$i.json 2>/dev/null
done
