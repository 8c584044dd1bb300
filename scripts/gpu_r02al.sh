# r02al: ELL (and HYB without a COO part) pinned spmv(m, x) following the upload
set -x
timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -p no:cacheprovider -k "pinned or follow or pageable or in_place or concurren or ell or ELL" > gpurun_out/al_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/al_pytest.log
for i in 1 2; do SOB_NO_CSR_FOLLOW=1 timeout 300 python scripts/e2e_quick.py 2>&1 | grep pinned | sed 's/^/oneshot /'; timeout 300 python scripts/e2e_quick.py 2>&1 | grep pinned | sed 's/^/follow /'; done
timeout 600 python scripts/ab_spmv.py after banded,hyb 2>&1 | tail -2
