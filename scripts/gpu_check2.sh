# Session-2 verification: tests, smoke, bench on the latest commits.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/c2_gpu.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/c2_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c2_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/c2_bench.log 2>&1; echo "bench rc=$?"
timeout 900 python scripts/spmv_sweep.py > gpurun_out/c2_sweep.log 2>&1; echo "sweep rc=$?"
tail -3 gpurun_out/c2_pytest_gpu.log
tail -1 gpurun_out/c2_bench.log
