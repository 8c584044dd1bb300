# r02 final evidence, pass 8 (final tree, 1 GPU): GPU suite, smoke, reference arm, e2e per format
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f8_pytest_gpu.log 2>&1; echo "suite rc=$? $(tail -1 gpurun_out/f8_pytest_gpu.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f8_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/f8_bench_ref.log 2>&1; echo "bench ref rc=$?"; tail -c 300 gpurun_out/f8_bench_ref.log
timeout 300 python scripts/e2e_formats.py 0,1,2,3,4,5 > gpurun_out/f8_e2e_formats.txt 2>&1; cat gpurun_out/f8_e2e_formats.txt
