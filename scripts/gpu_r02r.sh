# r02r: L2 prefetch-size qualifier on the streaming matrix loads (A/B builds)
for i in 1 2; do for v in base l2b256 l2b128; do AB_ROOT=build/ab_$v timeout 600 python scripts/ab_spmv.py $v banded,lap,hyb,rmat; done; done > gpurun_out/r_ab.txt 2>&1
cat gpurun_out/r_ab.txt
