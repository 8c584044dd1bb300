# r02an: pageable CSR / ELL follow A/B, 4 alternating rounds
for i in 1 2 3 4; do SOB_NO_CSR_FOLLOW=1 timeout 300 python scripts/e2e_quick.py 2>&1 | grep -E '^(1|3) pageable' | sed 's/^/staged /'; timeout 300 python scripts/e2e_quick.py 2>&1 | grep -E '^(1|3) pageable' | sed 's/^/follow /'; done
