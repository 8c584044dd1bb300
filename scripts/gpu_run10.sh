make -j8 >/dev/null 2>&1 || make -j8
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu10.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu10.log
timeout 1200 python scripts/config4.py --count 2000 --reps 20 --only profiles/config4_split_r01.json --model paper_2303_05098_b200/models/b200_forest.txt --out gpurun_out/config4_tuned_r01b.csv 2>&1 | tail -2
python scripts/config4_report.py gpurun_out/config4_tuned_r01b.csv
