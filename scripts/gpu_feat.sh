timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "feature or spread or full_size or random or structured or config1 or banded or rmat" 2>&1 | tail -2
timeout 600 python scripts/profile_features.py --ids 165 706 1692 521 --reps 5 2>&1 | grep "^id"
