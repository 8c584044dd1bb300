make -j8 >/dev/null 2>&1 || make -j8
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu9.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu9.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_banded9.csv python scripts/profile_spmv.py --workload banded --reps 1 > /dev/null 2>&1; echo "ncu rc=$?"
python scripts/ncu_summary.py launches gpurun_out/launches_banded9.csv | head -25
