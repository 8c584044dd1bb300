# r02t: CSR warp kernel at 2 CTAs/SM (97 regs: all 12 gathers in flight) vs 3 CTAs/SM (80 regs)
for i in 1 2; do for v in base b2; do AB_ROOT=build/ab_$v timeout 600 python scripts/ab_spmv.py $v rmat,unif,banded,hyb,lap; done; done > gpurun_out/t_ab.txt 2>&1
cat gpurun_out/t_ab.txt
