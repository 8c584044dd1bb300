# r02aa: follow-the-copy path for wide DIA windows (2-D stencils) -- parity + config-1 pinned e2e A/B
set -x
timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -p no:cacheprovider -k "pinned or follow or pageable or in_place or concurren" > gpurun_out/aa_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/aa_pytest.log
for i in 1 2; do SOB_NO_FOLLOW=1 timeout 300 python scripts/e2e_config1.py | sed 's/^/pipeline /'; timeout 300 python scripts/e2e_config1.py | sed 's/^/follow /'; done
timeout 300 python scripts/e2e_quick.py 2>&1 | grep '^2 '
