# r02z: tune plan times the all-direct sweep only when keys barely repeat
set -x
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_tuner_corpus.py -p no:cacheprovider -k "tune or feature or corpus" > gpurun_out/z_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/z_pytest.log
timeout 600 python scripts/tune_rmat_probe.py 2>&1 | sed "s/^/auto /"
python - <<'PY'
import time, sys
sys.path.insert(0, '.')
import paper_2303_05098_b200 as P, bench
from paper_2303_05098_b200 import synth
f = P.DeviceForest(bench.forest_ff())
csr = synth.banded(4_000_000, 13, seed=2)
d = P.DeviceMatrix.csr(csr.nrows, csr.ncols, csr.row_ptr, csr.col, csr.val)
t = time.perf_counter(); P.tune_ml(d, f); print("banded first tune_ml (plan build) %.1f ms" % ((time.perf_counter() - t) * 1e3))
PY
timeout 600 python scripts/tune_cost_probe.py > gpurun_out/z_tune_cost.txt 2>&1; tail -1 gpurun_out/z_tune_cost.txt
