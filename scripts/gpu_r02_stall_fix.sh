# Staging-pool stall fix (1 GPU): the failed-allocation stress test, the host-buffer set 6x, then the whole GPU suite
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "failed_allocation" > gpurun_out/sf_stress.log 2>&1; echo "stress rc=$? $(tail -1 gpurun_out/sf_stress.log)"
for i in 1 2 3 4 5 6; do
  timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "coo or pinned or follow or hdc or host" > gpurun_out/sf_set_$i.log 2>&1; echo "set $i rc=$? $(tail -1 gpurun_out/sf_set_$i.log)"
done
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/sf_pytest_gpu.log 2>&1; echo "suite rc=$? $(tail -1 gpurun_out/sf_pytest_gpu.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sf_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --no-config4 > gpurun_out/sf_bench.log 2>&1; echo "bench rc=$?"; tail -c 300 gpurun_out/sf_bench.log
