# r02aw: COO CONT (rows <= 32) forced on config 2 (SOB_COO_CONT=1) vs the size gate (records there)
for i in 1 2; do
SOB_COO_CONT=1 timeout 600 python scripts/ab_spmv.py cont_forced banded,unif 2>&1 | tail -2
timeout 600 python scripts/ab_spmv.py gated banded,unif 2>&1 | tail -2
done
