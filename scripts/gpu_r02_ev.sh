# r02 evidence run (1 GPU): GPU tests, smoke, bench (both arms), access-pattern
# probes, pageable e2e A/B, sanitizers over the full driver, ncu launch list.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/ev2_gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ev2_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/ev2_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev2_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/ev2_bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/ev2_bench_ref.log 2>&1; echo "bench ref rc=$?"
LAB_ONLY_PROD=1 LAB_GATHER=1 LAB_TRAFFIC=1 LAB_PEAK=6539.5 timeout 900 ./build/lab band,rmat,lap > gpurun_out/ev2_lab.log 2>&1; echo "lab rc=$?"
timeout 300 python scripts/e2e_quick.py > gpurun_out/ev2_e2e.log 2>&1; SOB_NO_NT_COPY=1 timeout 300 python scripts/e2e_quick.py 2>&1 | sed 's/^/nont /' >> gpurun_out/ev2_e2e.log; echo "e2e rc=$?"
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t $( [ $t = memcheck ] && echo --leak-check no ) python scripts/sanitize_driver.py > gpurun_out/ev2_sanitizer_$t.log 2>&1; echo "$t rc=$?"
done
timeout 900 compute-sanitizer --tool memcheck --target-processes all python scripts/sanitize_driver.py dist2 > gpurun_out/ev2_sanitizer_memcheck_dist2.log 2>&1; echo "dist2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 800 --csv --log-file gpurun_out/ev2_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-config4 --no-config5 > gpurun_out/ev2_bench_under_ncu.log 2>&1; echo "ncu list rc=$?"
tail -c 600 gpurun_out/ev2_bench.log
tail -c 400 gpurun_out/ev2_bench_ref.log
grep -h "ERROR SUMMARY" gpurun_out/ev2_sanitizer_*.log
