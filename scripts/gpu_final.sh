# End-of-round evidence run (1 GPU): tests, bench (both arms), ncu launch list
# of the bench, full capture of the headline kernel, per-format sweep,
# configs 4 and 5.  Everything lands in gpurun_out/.
set -x
make -j8 >/dev/null 2>&1 || make -j8
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/final_gpu.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/final_bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/final_bench_ref.log 2>&1; echo "bench ref rc=$?"
timeout 900 python scripts/spmv_sweep.py > gpurun_out/final_sweep.log 2>&1; echo "sweep rc=$?"
timeout 900 python scripts/config5.py --g 512 --iters 20 > gpurun_out/final_config5.log 2>&1; echo "c5 rc=$?"
timeout 1200 python scripts/config4.py --count 2000 --reps 20 --only profiles/config4_split_r01.json --model paper_2303_05098_b200/models/b200_forest.txt --out gpurun_out/final_config4_tuned.csv > gpurun_out/final_config4.log 2>&1; echo "c4 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/final_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/final_bench_under_ncu.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dia_kernel -s 2 -c 1 -o gpurun_out/final_full_dia python scripts/profile_spmv.py --workload banded --reps 2 --formats 5 > /dev/null 2>&1; echo "ncu full dia rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:csr_warp_kernel -s 1 -c 1 -o gpurun_out/final_full_csr python scripts/profile_spmv.py --workload banded --reps 1 --formats 1 > /dev/null 2>&1; echo "ncu full csr rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:coo_chunk_kernel -s 1 -c 1 -o gpurun_out/final_full_coo python scripts/profile_spmv.py --workload rmat --reps 1 --formats 0 > /dev/null 2>&1; echo "ncu full coo rc=$?"
tail -1 gpurun_out/final_bench.log
tail -1 gpurun_out/final_bench_ref.log
