# r02 final evidence (final tree, pass 7) (1 GPU): GPU suite, smoke, bench (both arms), N=2 / N=4 bench on one GPU,
# ncu launch list of the bench, full capture of the headline kernel, sanitizers over the full driver,
# config-4 tune cost probe, config-3 tune, host-buffer e2e
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/f7_gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f7_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/f7_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f7_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/f7_bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/f7_bench_ref.log 2>&1; echo "bench ref rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/f7_bench_n2.log 2>&1; echo "bench n2 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29553 bench.py --gpus 4 --steps 5 --warmup 3 --no-config4 > gpurun_out/f7_bench_n4.log 2>&1; echo "bench n4 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 800 --csv --log-file gpurun_out/f7_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-config4 --no-config5 --no-other-configs > gpurun_out/f7_bench_under_ncu.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dia_kernel -s 2 -c 1 -o gpurun_out/f7_full_dia python scripts/profile_spmv.py --workload banded --reps 3 --formats 2 > /dev/null 2>&1; echo "ncu dia rc=$?"
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t $( [ $t = memcheck ] && echo --leak-check no ) python scripts/sanitize_driver.py > gpurun_out/f7_sanitizer_$t.log 2>&1; echo "$t rc=$?"
done
timeout 900 compute-sanitizer --tool memcheck --target-processes all python scripts/sanitize_driver.py dist2 > gpurun_out/f7_sanitizer_memcheck_dist2.log 2>&1; echo "dist2 rc=$?"
timeout 600 python scripts/tune_cost_probe.py > gpurun_out/f7_tune_cost.txt 2>&1; echo "tune probe rc=$?"
timeout 600 python scripts/tune_rmat_probe.py > gpurun_out/f7_tune_rmat.txt 2>&1; echo "tune rmat rc=$?"
timeout 600 python scripts/e2e_quick.py > gpurun_out/f7_e2e.txt 2>&1; for i in 1 2; do timeout 300 ./build/e2e_api 30 3; done >> gpurun_out/f7_e2e.txt 2>&1
tail -c 600 gpurun_out/f7_bench.log
tail -c 400 gpurun_out/f7_bench_ref.log
grep -h "ERROR SUMMARY\|RACECHECK SUMMARY" gpurun_out/f7_sanitizer_*.log
tail -1 gpurun_out/f7_tune_cost.txt
cat gpurun_out/f7_tune_rmat.txt
timeout 300 python scripts/e2e_formats.py 0,1,2,3,4,5 > gpurun_out/f7_e2e_formats.txt 2>&1
bash scripts/gpu_r02aj.sh > gpurun_out/f7_c4.log 2>&1
