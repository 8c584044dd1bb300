# r02ap: debug HYB (with a COO part) follow path
for a in "600000 pinned" "600000 pageable" "4000000 pinned" "4000000 pageable"; do
  echo "== $a"; timeout 120 python scripts/hyb_follow_debug.py $a 2>&1 | tail -25
done
echo "== coo off"; SOB_NO_COO_FOLLOW=1 timeout 120 python scripts/hyb_follow_debug.py 600000 pinned 2>&1 | tail -5
