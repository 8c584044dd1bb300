timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/it_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/it_pytest.log
LAB_ONLY_PROD=1 LAB_PEAK=6539.5 timeout 600 ./build/lab band,lap,rmat > gpurun_out/it_lab.log 2>&1; echo "lab rc=$?"
grep "CSR\|HDC\|n=" gpurun_out/it_lab.log
timeout 900 python scripts/convert_bench.py 2>&1 | tail -4
