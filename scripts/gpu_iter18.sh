timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/it_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/it_pytest.log
timeout 900 python scripts/convert_bench.py 2>&1 | tail -4
