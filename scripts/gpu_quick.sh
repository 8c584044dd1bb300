# Iteration helper (1 GPU): the GPU test suite and the product kernels on
# configs 1-3 (scripts/spmv_lab.cu, product rows only).
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/q_pytest.log
LAB_ONLY_PROD=1 LAB_PEAK=$(python -c "import json;print(json.load(open('MEASURED_PEAKS.json'))['hbm_gbs'])") \
  timeout 600 ./build/lab band,lap,rmat > gpurun_out/q_lab.log 2>&1; echo "lab rc=$?"
cat gpurun_out/q_lab.log
