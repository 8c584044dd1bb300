# r02 final (2): GPU suite, smoke, bench on the final tree
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g2_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/g2_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g2_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/g2_bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/g2_bench_ref.log 2>&1; echo "bench ref rc=$?"
tail -c 400 gpurun_out/g2_bench_ref.log
