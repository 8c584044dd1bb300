# r02ab: config-1 pinned e2e, follow vs chunk pipeline, 4 alternating rounds
for i in 1 2 3 4; do SOB_NO_FOLLOW=1 timeout 300 python scripts/e2e_config1.py | sed 's/^/pipeline /'; timeout 300 python scripts/e2e_config1.py | sed 's/^/follow /'; done
