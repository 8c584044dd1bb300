# r02c evidence (HEAD 29779ab, fresh container rebuild) run (1 GPU): GPU tests, smoke, bench (both arms)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/ev4_gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ev4_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/ev4_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev4_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/ev4_bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/ev4_bench_ref.log 2>&1; echo "bench ref rc=$?"
tail -c 600 gpurun_out/ev4_bench.log
tail -c 400 gpurun_out/ev4_bench_ref.log
