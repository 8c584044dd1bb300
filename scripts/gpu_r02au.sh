# r02au: COO rows finished by the chunk that starts them (CONT: no records, no fix-up) vs records + coo_fixup (SOB_NO_COO_CONT=1)
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/au_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/au_pytest.log; grep -E "^FAILED|^E " gpurun_out/au_pytest.log | head -20
for i in 1 2 3; do
  SOB_NO_COO_CONT=1 timeout 600 python scripts/ab_spmv.py records lap,banded,hyb,rmat 2>&1 | tail -4
  timeout 600 python scripts/ab_spmv.py cont lap,banded,hyb,rmat 2>&1 | tail -4
done
for i in 1 2; do
  SOB_NO_COO_CONT=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-config4 --no-config5 --no-cpu-baseline > gpurun_out/au_bench_records_$i.json 2>/dev/null
  timeout 600 python bench.py --steps 20 --warmup 5 --no-config4 --no-config5 --no-cpu-baseline > gpurun_out/au_bench_cont_$i.json 2>/dev/null
done
timeout 300 python scripts/e2e_formats.py 0,4 2>&1 | sed 's/^/e2e /'
