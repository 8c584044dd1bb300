timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/it_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/it_pytest.log
LAB_ONLY_PROD=1 LAB_PEAK=6539.5 timeout 600 ./build/lab band,rmat > gpurun_out/it_lab.log 2>&1; echo "lab rc=$?"
cat gpurun_out/it_lab.log
for k in csr_long_pieces csr_warp_kernel coo_warp_kernel; do
LAB_ONLY_PROD=1 LAB_REPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 2 -c 1 -o gpurun_out/rmat_$k ./build/lab rmat > /dev/null 2>&1; echo "ncu $k rc=$?"
done
