# r02bc: pinned CSR chunk pipeline with 16 chunks (vs 8 in r02bb)
for i in 1 2 3; do
  timeout 300 python scripts/e2e_formats.py 1 2>&1 | grep pinned | sed 's/^/k16 /'
done
