timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/feat_small_warm.csv python scripts/profile_features.py --ids 165 1692 --reps 3 > /dev/null 2>&1; echo "ncu rc=$?"
timeout 600 python scripts/profile_features.py --ids 165 706 1692 521 --reps 5 2>&1 | grep "^id"
