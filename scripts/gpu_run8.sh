make -j8 >/dev/null 2>&1 || make -j8
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "stencil27 or structured or rmat or laplacian or banded" > gpurun_out/pytest_gpu8.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu8.log
timeout 900 python scripts/config5.py --g 512 --iters 20 2>&1 | tail -2
timeout 900 python scripts/config5.py --g 256 --iters 20 2>&1 | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_r01.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dia_kernel -s 2 -c 1 -o gpurun_out/full_dia_bench_r01 python scripts/profile_spmv.py --workload banded --reps 2 --formats 5 > /dev/null 2>&1; echo "ncu full rc=$?"
