make -j8 >/dev/null 2>&1 || make -j8
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu5.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu5.log
timeout 900 python scripts/spmv_sweep.py 2>&1 | tail -40
