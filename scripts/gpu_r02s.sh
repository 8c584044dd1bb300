# r02s: CSR on R-MAT -- launch list and full captures of the warp kernel and the long-row pieces
set -x
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s_launches_csr_rmat.csv python scripts/profile_spmv.py --workload rmat --reps 3 --formats 1 > /dev/null 2>&1; echo "list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:csr_warp_kernel -s 1 -c 1 -o gpurun_out/s_full_csr_warp_rmat python scripts/profile_spmv.py --workload rmat --reps 1 --formats 1 > /dev/null 2>&1; echo "full warp rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:csr_long_pieces -s 1 -c 1 -o gpurun_out/s_full_csr_pieces_rmat python scripts/profile_spmv.py --workload rmat --reps 1 --formats 1 > /dev/null 2>&1; echo "full pieces rc=$?"
