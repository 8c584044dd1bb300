# r02ba: HDC with both parts follows the upload (DIA follow kernel, then the CSR part accumulating, into device y)
set -x
python - <<'PY'
import sys; sys.path.insert(0, '.')
import paper_2303_05098_b200 as P
from paper_2303_05098_b200 import synth
for args in ((600_000, 8, 40, 50, 6), (4_000_000, 16, 160, 100, 6)):
    c = synth.hyb_skewed(*args[:4], seed=args[4])
    m = P.DeviceMatrix.csr(c.nrows, c.ncols, c.row_ptr, c.col, c.val).convert(5)
    h = m.download()
    print("hdc parts", args, {k: (v.shape if hasattr(v, "shape") else v) for k, v in h.items() if k in ("offsets", "col", "values")})
PY
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "pinned or follow or pageable or concurren or in_place or hdc or HDC" > gpurun_out/ba_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ba_pytest.log; grep -E "^E |FAILED" gpurun_out/ba_pytest.log | head
for i in 1 2 3; do
  SOB_NO_HDC_FOLLOW=1 timeout 300 python scripts/e2e_formats.py 5 2>&1 | sed 's/^/before /'
  timeout 300 python scripts/e2e_formats.py 5 2>&1 | sed 's/^/after /'
done
