timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/it_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/it_pytest.log
timeout 600 python scripts/profile_features.py --ids 877 1843 555 165 706 1692 521 --reps 5 2>&1 | grep "^id"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/feat_small_warm.csv python scripts/profile_features.py --ids 1692 706 --reps 2 > /dev/null 2>&1; echo "ncu rc=$?"
