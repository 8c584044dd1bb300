# r02u: COO grid: persistent (num_sms x 3 CTAs) vs 4x / 64x more CTAs (fewer chunks per warp)
for i in 1 2; do for v in base g4 g64; do AB_ROOT=build/ab_$v timeout 600 python scripts/ab_spmv.py $v lap,banded,rmat,hyb; done; done > gpurun_out/u_ab.txt 2>&1
cat gpurun_out/u_ab.txt
