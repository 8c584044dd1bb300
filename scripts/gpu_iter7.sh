LAB_ONLY_PROD=1 LAB_COO=1 LAB_PEAK=6539.5 timeout 600 ./build/lab band,rmat,lap > gpurun_out/it_lab.log 2>&1; echo "lab rc=$?"
grep -v "^  prod" gpurun_out/it_lab.log
