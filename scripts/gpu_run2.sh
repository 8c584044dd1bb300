set -x
make -j8 >/dev/null 2>&1 || make -j8
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench2.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/bench2.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_banded.csv python scripts/profile_spmv.py --workload banded > gpurun_out/prof_banded.log 2>&1; echo "ncu rc=$?"
tail -20 gpurun_out/prof_banded.log
