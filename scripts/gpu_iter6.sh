COPY_PROBE=1 python scripts/e2e_probe.py
for c in 1 4 8 32; do SOB_PIPE_CHUNKS=$c python scripts/e2e_probe.py; done
LAB_ONLY_PROD=1 LAB_COO=1 LAB_PEAK=6539.5 timeout 600 ./build/lab band,rmat > gpurun_out/it_lab.log 2>&1; echo "lab rc=$?"
grep -v "^  prod" gpurun_out/it_lab.log
