make -j8 >/dev/null 2>&1 || make -j8
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu6.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu6.log
timeout 2400 python scripts/config4.py --count 2000 --reps 20 --out gpurun_out/config4_profile_2000.csv 2>&1 | tail -3
