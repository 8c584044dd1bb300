# Evidence run (1 GPU): tests, smoke, bench (both arms), per-format sweep,
# config 5, ncu launch list of the bench, full captures of the SpMV kernels.
# Everything lands in gpurun_out/ev_*.
set -x
make -j8 >/dev/null 2>&1 || make -j8
make tools >/dev/null 2>&1 || make tools
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/ev_gpu.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ev_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/ev_bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/ev_bench_ref.log 2>&1; echo "bench ref rc=$?"
LAB_ONLY_PROD=1 LAB_PEAK=$(python -c "import json;print(json.load(open('MEASURED_PEAKS.json'))['hbm_gbs'])") timeout 600 ./build/lab band,lap,rmat > gpurun_out/ev_lab.log 2>&1; echo "lab rc=$?"
timeout 900 python scripts/config5.py --g 512 --iters 20 > gpurun_out/ev_config5.log 2>&1; echo "c5 rc=$?"
timeout 900 python scripts/convert_bench.py > gpurun_out/ev_convert.log 2>&1; echo "convert rc=$?"
timeout 1500 python scripts/config4.py --count 2000 --reps 20 --only profiles/config4_split_r01b.json --model paper_2303_05098_b200/models/b200_forest.txt --out gpurun_out/ev_c4_tuned.csv > gpurun_out/ev_c4.log 2>&1; echo "c4 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/ev_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev_bench_under_ncu.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dia_kernel -s 2 -c 1 -o gpurun_out/ev_full_dia python scripts/profile_spmv.py --workload banded --reps 2 --formats 5 > /dev/null 2>&1; echo "ncu dia rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:csr_warp_kernel -s 1 -c 1 -o gpurun_out/ev_full_csr python scripts/profile_spmv.py --workload banded --reps 1 --formats 1 > /dev/null 2>&1; echo "ncu csr rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:coo_warp_kernel -s 1 -c 1 -o gpurun_out/ev_full_coo_band python scripts/profile_spmv.py --workload banded --reps 1 --formats 0 > /dev/null 2>&1; echo "ncu coo band rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:coo_warp_kernel -s 1 -c 1 -o gpurun_out/ev_full_coo_rmat python scripts/profile_spmv.py --workload rmat --reps 1 --formats 0 > /dev/null 2>&1; echo "ncu coo rmat rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ell_kernel -s 1 -c 1 -o gpurun_out/ev_full_ell python scripts/profile_spmv.py --workload banded --reps 1 --formats 3 > /dev/null 2>&1; echo "ncu ell rc=$?"
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches_rmat_features_convert.csv python scripts/profile_rmat_path.py > /dev/null 2>&1; echo "ncu rmat path rc=$?"
timeout 600 python scripts/e2e_probe.py > gpurun_out/ev_e2e.log 2>&1; SOB_NO_ZERO_COPY=1 timeout 600 python scripts/e2e_probe.py >> gpurun_out/ev_e2e.log 2>&1; echo "e2e rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dia_zc_kernel -c 1 -o gpurun_out/ev_full_dia_zc python scripts/e2e_probe.py > /dev/null 2>&1; echo "ncu zc rc=$?"
tail -1 gpurun_out/ev_bench.log
tail -1 gpurun_out/ev_bench_ref.log
tail -3 gpurun_out/ev_config5.log
