# r02at: ncu full capture of coo_warp_kernel on config 1 (Laplacian 1000^2)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:coo_warp_kernel -s 2 -c 1 -o gpurun_out/at_coo_lap python scripts/profile_spmv.py --workload laplacian --reps 3 --formats 0 > gpurun_out/at_ncu.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/at_launches_lap.csv python scripts/profile_spmv.py --workload laplacian --reps 3 > /dev/null 2>&1; echo "list rc=$?"
