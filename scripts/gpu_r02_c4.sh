# r02: config-4 batch profiling on the B200 (2000 matrices, 20 reps, twins
# recorded, twin-equalised wire CSVs for the reference trainer)
set -x
timeout 2400 python scripts/config4.py --count 2000 --reps 20 --out gpurun_out/r02_c4_profile.csv --ref-csv gpurun_out/r02_c4_wire > gpurun_out/r02_c4.log 2>&1; echo "c4 rc=$?"
tail -3 gpurun_out/r02_c4.log
