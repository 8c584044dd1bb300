# r02e: A/B of y growth steps in the C++ API e2e (same box, alternating)
for r in 1 2 3; do for s in 1 4 16 64; do echo "== SOB_Y_STEPS=$s"; SOB_Y_STEPS=$s timeout 300 ./build/e2e_api 30 3 | cut -c1-260; done; done > gpurun_out/e_ab.txt 2>&1
cat gpurun_out/e_ab.txt
