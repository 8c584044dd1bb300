set -x
make -j8 >/dev/null 2>&1 || make -j8
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/g1_pytest.log 2>&1; echo "pytest rc=$?"
timeout 600 python scripts/profile_features.py --ids 877 543 13 7 --reps 5 > gpurun_out/g1_feat.log 2>&1; echo "feat rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g1_feat_launches.csv python scripts/profile_features.py --ids 877 543 --reps 1 > /dev/null 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/g1_pytest.log; cat gpurun_out/g1_feat.log
