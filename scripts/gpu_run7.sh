make -j8 >/dev/null 2>&1 || make -j8
timeout 1200 python scripts/config4.py --count 2000 --reps 20 --only profiles/config4_split_r01.json --model paper_2303_05098_b200/models/b200_forest.txt --out gpurun_out/config4_tuned_r01.csv 2>&1 | tail -3
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/bench7.log 2>&1; echo "bench rc=$?"; tail -2 gpurun_out/bench7.log
