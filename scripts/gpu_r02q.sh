# r02q: injected-tool detection for the follow path; bench launch list under ncu; sanitizer on the pinned case
set -x
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 800 --csv --log-file gpurun_out/q_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-config4 --no-config5 --no-other-configs > gpurun_out/q_bench_under_ncu.log 2>&1; echo "ncu list rc=$?"
timeout 900 compute-sanitizer --tool memcheck --leak-check no python scripts/sanitize_driver.py --quick > gpurun_out/q_memcheck.log 2>&1; echo "memcheck rc=$?"; grep -h "ERROR SUMMARY" gpurun_out/q_memcheck.log
timeout 300 python scripts/e2e_quick.py 2>&1 | grep '^2 '
