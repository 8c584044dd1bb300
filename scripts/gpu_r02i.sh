# r02i: RED.ADD for HDC's CSR part too (redcsr) vs red2 (HYB only)
set -x
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_full_size.py -p no:cacheprovider -k "hdc or HDC or hyb or HYB or random or switch or pageable" > gpurun_out/i_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/i_pytest.log
for i in 1 2; do for v in red2 redcsr; do AB_ROOT=build/ab_$v timeout 600 python scripts/ab_spmv.py $v hyb,banded,lap; done; done > gpurun_out/i_ab.txt 2>&1
cat gpurun_out/i_ab.txt
