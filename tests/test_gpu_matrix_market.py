"""read_matrix_market / write_matrix_market against the
reference's own implementation (ingest.cpp:135-224, compiled in place): the
same canonical COO bit for bit, or the same error type AND message (path and
line number included) for every malformed input -- the host-parallel parser
must report the first error in FILE order, also when the slices are parsed
by different threads (the large-file cases).  Reference test cases:
test_ingest.cpp:62-156."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HDR = "%%MatrixMarket matrix coordinate real general\n"


@pytest.fixture(scope="module")
def R():
    import oracle

    if not oracle.refpipe_available():
        pytest.skip("reference pipeline not built (oracle/Makefile refpipe)")
    return oracle


def _ours(so, path):
    try:
        m = so.DeviceMatrix.read_matrix_market(path)
    except (so.ParseError, so.UnsupportedFormat, so.IndexOutOfRange) as e:
        return type(e).__name__, str(e)
    return "ok", m.download()


def _same(so, R, path):
    want = R.ref_read_matrix_market(path)
    got = _ours(so, path)
    assert got[0] == want[0], (path, got, want)
    if want[0] != "ok":
        assert got[1] == want[1]
        return want
    g, w = got[1], want[1]
    assert (g["nrows"], g["ncols"]) == (w["nrows"], w["ncols"])
    for k in ("row", "col", "val"):
        assert np.array_equal(np.asarray(g[k]), w[k]), k
    return want


CASES = {
    # test_ingest.cpp:51-66 worked example
    "worked": HDR + "% the worked example\n3 3 5\n1 1 1\n1 3 2\n2 2 3\n3 1 4\n3 3 5\n",
    "sym": "%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 5\n2 1 7\n",
    "pattern": "%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 2\n2 1\n",
    "integer": "%%MatrixMarket matrix coordinate integer general\n1 2 1\n1 2 -3\n",
    "complex": "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "array": "%%MatrixMarket matrix array real general\n1 1\n1\n",
    "skew": "%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n2 1 1\n",
    "short": HDR + "3 3 5\n1 1 1\n1 3 2\n2 2 3\n3 1 4\n",
    "long": HDR + "2 2 1\n1 1 1\n2 2 2\n",
    "bad_int": HDR + "2 2 1\n1 x 1\n",
    "oob": HDR + "2 2 1\n3 1 1\n",
    # beyond the reference suite: every branch of ingest.cpp:135-208
    "empty": "",
    "no_banner": "%%Matrix matrix coordinate real general\n1 1 1\n1 1 1\n",
    "object": "%%MatrixMarket vector coordinate real general\n1 1 1\n1 1 1\n",
    "no_dims": HDR + "% only comments\n\n",
    "dims_tokens": HDR + "2 2\n1 1 1\n",
    "dims_bad": HDR + "2 two 1\n1 1 1\n",
    "dims_neg": HDR + "-2 2 1\n1 1 1\n",
    "sym_rect": "%%MatrixMarket matrix coordinate real symmetric\n2 3 1\n1 1 1\n",
    "tokens": HDR + "2 2 2\n1 1 1 9\n2 2 2\n",
    "bad_val": HDR + "2 2 1\n1 1 abc\n",
    "long_and_bad": HDR + "2 2 1\n1 1 1\n2 x 2\n",
    "crlf": HDR.replace("\n", "\r\n") + "2 2 2\r\n\r\n% c\r\n1 1 1.5\r\n2 2 -0.25\r\n",
    "tabs_no_eol": HDR + "2\t2\t2\n1\t2\t1e-3\n2 1 +3",
    "dup": HDR + "2 2 3\n1 1 1\n1 1 2\n2 2 4\n",
    "pattern_extra": "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 2 3\n",
    "upper": "%%MATRIXMARKET MATRIX COORDINATE REAL GENERAL\n1 1 1\n1 1 1\n",
    "upper2": "%%MatrixMarket MATRIX Coordinate REAL General\n1 1 1\n1 1 1\n",
    "zero": HDR + "0 0 0\n",
    "inf": HDR + "1 2 2\n1 1 inf\n1 2 -1e308\n",
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_matches_reference(so, R, tmp_path, name):
    p = tmp_path / f"{name}.mtx"
    p.write_bytes(CASES[name].encode())
    _same(so, R, p)


def _big(n, nnz, rng):
    r = rng.integers(1, n + 1, nnz)
    c = rng.integers(1, n + 1, nnz)
    v = rng.uniform(-2, 2, nnz)
    return [f"{a} {b} {x!r}\n" for a, b, x in zip(r, c, v)]


@pytest.mark.parametrize("kind", ["ok", "late_error", "two_errors", "overflow_late", "underflow"])
def test_large_files_multithreaded(so, R, tmp_path, kind):
    """~6 MB bodies (several host slices): the first error in file order wins."""
    rng = np.random.default_rng(7)
    n, nnz = 50_000, 200_000
    lines = _big(n, nnz, rng)
    declared = nnz
    if kind == "late_error":
        lines[190_000] = "5 bad 1\n"
    elif kind == "two_errors":
        lines[150_000] = f"{n + 1} 1 1\n"   # IndexOutOfRange, later slice
        lines[60_000] = "1 2\n"             # token count, earlier slice: this one wins
    elif kind == "overflow_late":
        declared = 170_000
        lines[185_000] = "x y z\n"          # after the overflow point: overflow wins
    elif kind == "underflow":
        declared = nnz + 3
    p = tmp_path / f"{kind}.mtx"
    p.write_text(HDR + f"% {kind}\n{n} {n} {declared}\n" + "".join(lines))
    _same(so, R, p)


def test_write_is_byte_identical_and_round_trips(so, R, O, tmp_path):
    rng = O.Rng(61)  # test_ingest.cpp:147-156
    for trial in range(12):
        coo = rng.random_coo(40)
        d = so.DeviceMatrix.coo(coo["nrows"], coo["ncols"], coo["row"], coo["col"], coo["val"])
        ours, ref = tmp_path / f"o{trial}.mtx", tmp_path / f"r{trial}.mtx"
        d.write_matrix_market(ours)
        R.ref_write_matrix_market(ref, coo)
        assert ours.read_bytes() == ref.read_bytes()
        back = so.DeviceMatrix.read_matrix_market(ours).download()
        for k in ("row", "col", "val"):
            assert np.array_equal(np.asarray(back[k]), np.asarray(coo[k]))
