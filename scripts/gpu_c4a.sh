make -j8 >/dev/null 2>&1 || make -j8
mkdir -p gpurun_out
timeout 2400 python scripts/config4.py --count 600 --reps 20 --out gpurun_out/config4_profile_r1.csv 2>&1 | tail -5
