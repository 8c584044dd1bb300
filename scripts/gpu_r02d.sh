# r02d: progressive-y C++ API e2e, N>1 checksum protocol (2 ranks sharing the GPU), per-format CPU baseline
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "pageable or spmv_new or concurren" > gpurun_out/d_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/d_pytest.log
for i in 1 2; do timeout 300 ./build/e2e_api 20 3; done > gpurun_out/d_e2e_api.txt 2>&1
SOB_STAGE_TRACE=1 timeout 300 ./build/e2e_api 6 2 > gpurun_out/d_e2e_trace.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-config4 > gpurun_out/d_bench2.log 2>&1; echo "bench2 rc=$?"
timeout 900 python bench.py --steps 10 --warmup 3 --no-other-configs --no-config4 --no-cpu-baseline > gpurun_out/d_bench1.log 2>&1; echo "bench1 rc=$?"
timeout 1500 python scripts/cpu_baseline.py > gpurun_out/d_cpu_baseline.json 2> gpurun_out/d_cpu_baseline.err; echo "cpu rc=$?"
cat gpurun_out/d_e2e_api.txt | cut -c1-400
grep -h checksum gpurun_out/d_bench2.log | cut -c1-300
