# r02av: COO CONT gated on size and rows <= 32; parity of both COO paths + follow/pinned subset
set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "coo or COO or hyb or HYB or pinned or follow or pageable" > gpurun_out/av_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/av_pytest.log; grep -E "^FAILED|^E " gpurun_out/av_pytest.log | head
for i in 1 2; do
SOB_NO_COO_CONT=1 timeout 600 python scripts/ab_spmv.py records lap,hyb 2>&1 | tail -2
timeout 600 python scripts/ab_spmv.py gated lap,banded,hyb 2>&1 | tail -3
done
