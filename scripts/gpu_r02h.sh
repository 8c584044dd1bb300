# r02h: HYB's COO part accumulating with RED.ADD.F64 (2 or 3 CTAs/SM) vs the load+add kernel (base)
set -x
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_full_size.py -p no:cacheprovider -k "hyb or HYB or rmat or random or switch or coo" > gpurun_out/h_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/h_pytest.log
for i in 1 2; do for v in base red2 red3; do AB_ROOT=build/ab_$v timeout 600 python scripts/ab_spmv.py $v rmat,unif,hyb; done; done > gpurun_out/h_ab.txt 2>&1
cat gpurun_out/h_ab.txt
