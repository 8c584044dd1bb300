"""GPU: the reference's OWN unit and acceptance suites (proj/tests/test_formats.cpp,
test_spmv.cpp, test_features.cpp, test_model.cpp, test_tuners.cpp; 59 test
cases), compiled unmodified against this repo's C++ API
(include/sparseoracle/*.hpp over the sm_100a library) by `make reftests`,
with tests/support/doctest_shim standing in for the absent vendored doctest.
Every case must pass: that is the drop-in claim for the hot path.
"""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(REPO, "build", "reftests")
# + the Matrix Market cases of test_ingest.cpp restated in tests/support/cpp,
# and concurrent readers of one lazily materialised matrix
SUITES = ["formats", "spmv", "features", "model", "tuners", "matrix_market", "concurrency",
          # the reference's acceptance suite (10 criteria) and its pipeline /
          # trainer suites: reference code above the path (make refaccept),
          # every hot-path call and every Matrix Market read through this repo
          "acceptance", "pipeline", "trainer", "ingest"]


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite(suite):
    exe = os.path.join(BIN, suite if suite == "acceptance" else f"test_{suite}")
    if not os.path.exists(exe):
        if os.path.isdir("/root/reference/proj/tests"):
            subprocess.run(["make", "-C", REPO, "reftests"], check=True, capture_output=True)
        else:
            pytest.skip("reference suites not built here and /root/reference absent")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=900, cwd=REPO)
    print(p.stdout)
    print(p.stderr[-4000:])
    assert "[FAIL]" not in p.stdout, p.stderr[-4000:]
    assert p.returncode == 0
