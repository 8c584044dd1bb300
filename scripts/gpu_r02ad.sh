# r02ad: host copy pool size (SOB_HOST_THREADS) for the pageable / C++ API paths: 16 (= hardware threads) vs 15 vs 12 vs 8
for i in 1 2; do for t in 16 15 12 8; do
  echo "== threads $t"; SOB_HOST_THREADS=$t timeout 300 python scripts/e2e_quick.py 2>&1 | grep -E '^2 (pageable|fresh)'
  SOB_HOST_THREADS=$t timeout 300 ./build/e2e_api 30 3 | cut -c1-200
done; done
