make -j8 >/dev/null 2>&1 || make -j8
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu3.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu3.log
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench3.log 2>&1; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench3.log').read().strip().splitlines()[-1]);print(d['value'],d['roofline']['frac']);print(json.dumps(d['formats']))"
for k in csr_stream_kernel coo_chunk_kernel dia_kernel; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o gpurun_out/full_$k python scripts/profile_spmv.py --workload banded --reps 1 > /dev/null 2>&1; echo "ncu $k rc=$?"
done
ls -la gpurun_out/
