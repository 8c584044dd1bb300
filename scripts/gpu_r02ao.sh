# r02ao: COO (and HYB with a COO part) host-buffer spmv(m, x) following the upload of x into device y
set -x
for a in "600000 pinned" "4000000 pinned,pageable"; do timeout 120 python scripts/hyb_follow_debug.py $a 2>&1 | tail -8; done
timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -p no:cacheprovider -k "pinned or follow or pageable or in_place or concurren or coo or COO or hyb" > gpurun_out/ao_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ao_pytest.log
for i in 1 2 3; do SOB_NO_COO_FOLLOW=1 timeout 300 python scripts/e2e_formats.py 2>&1 | sed 's/^/staged /'; timeout 300 python scripts/e2e_formats.py 2>&1 | sed 's/^/follow /'; done
