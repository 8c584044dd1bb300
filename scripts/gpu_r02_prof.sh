# r02: full ncu captures of the SpMV kernels on R-MAT (config 3) + sanitizer smoke
set -x
for spec in "csr_warp_kernel 1 csr" "coo_warp_kernel 0 coo" "ell_kernel 4 hyb_ell" "coo_warp_kernel 4 hyb_coo" "csr_warp_kernel 5 hdc"; do
  set -- $spec
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$1 -s 1 -c 1 -o gpurun_out/r02_full_$3_rmat python scripts/profile_spmv.py --workload rmat --reps 1 --formats $2 > /dev/null 2>&1; echo "ncu $3 rc=$?"
done
timeout 1200 compute-sanitizer --tool memcheck --leak-check no python scripts/sanitize_driver.py > gpurun_out/r02_memcheck.log 2>&1; echo "memcheck rc=$?"
tail -5 gpurun_out/r02_memcheck.log
