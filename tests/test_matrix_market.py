"""Matrix Market ingest: the library's C++ reader/writer behind the C ABI
(sssvd_mm_read / sssvd_mm_write) re-expressing proj/tests/test_matrix_market.cpp case by case,
then checked bit for bit against the oracle's restatement of matrix_market.hpp:34-119 on seeded
random files. Host-only: no GPU needed."""
import os

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import sssvd_oracle as orc


@pytest.fixture
def mm(tmp_path):
    from paper_2109_13655_b200 import sssvd

    def write(name, contents):
        p = tmp_path / name
        p.write_text(contents)
        return str(p)
    return sssvd, write


def test_array_format_column_major(mm):                       # test_matrix_market.cpp:30-40
    s, w = mm
    a = s.read_matrix_market(w("a.mtx", "%%MatrixMarket matrix array real general\n% a 2x2 example\n"
                                        "2 2\n1\n3\n2\n4\n"))
    assert not a.is_sparse()
    assert np.array_equal(a.to_dense(), np.array([[1.0, 2.0], [3.0, 4.0]]))


def test_coordinate_duplicates_summed(mm):                   # :42-55
    s, w = mm
    a = s.read_matrix_market(w("d.mtx", "%%MatrixMarket matrix coordinate real general\n3 2 3\n"
                                        "1 1 0.5\n1 1 0.5\n3 2 2.0\n"))
    assert a.is_sparse()
    d = a.to_dense()
    assert d[0, 0] == 1.0 and d[2, 1] == 2.0 and d.shape[0] == 3


def test_symmetric_coordinate_expands(mm):                   # :57-68
    s, w = mm
    d = s.read_matrix_market(w("s.mtx", "%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n"
                                        "1 1 5\n2 1 3\n")).to_dense()
    assert d[0, 1] == 3.0 and d[1, 0] == 3.0 and d[0, 0] == 5.0


def test_pattern_and_complex_rejected(mm):                   # :70-78
    s, w = mm
    with pytest.raises(s.MatrixMarketError, match="unsupported field"):
        s.read_matrix_market(w("p.mtx", "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 1\n"))
    with pytest.raises(s.MatrixMarketError):
        s.read_matrix_market(w("c.mtx", "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1.0 0.0\n"))


def test_parse_error_carries_line_number(mm):                # :80-94
    s, w = mm
    with pytest.raises(s.MatrixMarketError, match=":5:"):
        s.read_matrix_market(w("b.mtx", "%%MatrixMarket matrix coordinate real general\n% comment\n2 2 2\n"
                                        "1 1 1.0\noops\n"))


def test_out_of_range_index_rejected(mm):                    # :96-99
    s, w = mm
    with pytest.raises(s.MatrixMarketError, match="index out of range"):
        s.read_matrix_market(w("o.mtx", "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n"))


def test_model_problem_round_trip_lossless(mm, tmp_path):    # :101-111
    s, _ = mm
    pm, *_ = orc.build_model(1, 60, 20, 7)
    a = s.ProblemMatrix.from_dense(pm.dense)
    path = str(tmp_path / "round.mtx")
    s.write_matrix_market(path, a, "round trip")
    back = s.read_matrix_market(path)
    assert np.array_equal(back.to_dense(), a.to_dense())     # 17 digits round-trip exactly
    assert open(path).read().splitlines()[1] == "% round trip"


def test_wide_round_trip_keeps_user_orientation(mm, tmp_path):   # :113-126
    s, _ = mm
    wide = np.array([[10.0 * (i + 1) + j for j in range(5)] for i in range(2)])
    p = s.ProblemMatrix.from_dense(wide)
    assert p.transposed()
    path = str(tmp_path / "wide.mtx")
    s.write_matrix_market(path, p, "")
    assert open(path).read().splitlines()[1] == "2 5"
    back = s.read_matrix_market(path)
    assert back.transposed()
    assert np.array_equal(back.to_dense(), wide.T)


def test_sparse_round_trip(mm, tmp_path):                    # :128-139
    s, _ = mm
    m = sp.lil_matrix((4, 3))
    m[0, 0] = 1.25
    m[3, 2] = -7.5e-13
    p = s.ProblemMatrix.from_sparse(m)
    path = str(tmp_path / "sp.mtx")
    s.write_matrix_market(path, p, "")
    back = s.read_matrix_market(path)
    assert back.is_sparse()
    assert np.array_equal(back.to_dense(), p.to_dense())


def test_missing_file(mm):                                   # :141-143
    s, _ = mm
    with pytest.raises(RuntimeError, match="cannot open"):
        s.read_matrix_market("/nonexistent/path.mtx")


@pytest.mark.parametrize("header,body,what", [
    ("%%MatrixMarket matrix coordinate real general", "", "missing size line"),
    ("%%MatrixMarket vector coordinate real general", "1 1 1\n", "not a MatrixMarket matrix header"),
    ("%%MatrixMarket matrix coordinate real hermitian", "1 1 1\n", "unsupported symmetry"),
    ("%%MatrixMarket matrix coordinate bogus general", "1 1 1\n", "unknown field 'bogus'"),
    ("%%MatrixMarket matrix weird real general", "1 1\n", "unknown format 'weird'"),
    ("%%MatrixMarket matrix array real general", "2 2\n1\n2\n3\n", "unexpected end of array data"),
    ("%%MatrixMarket matrix array real general", "0 2\n", "bad array size line"),
    ("%%MatrixMarket matrix coordinate real general", "2 2 2\n1 1 1\n", "unexpected end of coordinate data"),
    ("%%MatrixMarket matrix coordinate real general", "2 2 -1\n", "bad coordinate size line"),
    ("%%MatrixMarket matrix array real general", "1 1\ninf\n", "bad array value"),
])
def test_error_paths_match_oracle(mm, header, body, what):
    """Every reader error of matrix_market.hpp:36-112 with the oracle's text and line number."""
    s, w = mm
    path = w("e.mtx", header + "\n" + body)
    with pytest.raises(RuntimeError) as got:
        s.read_matrix_market(path)
    assert what in str(got.value)
    if what != "bad array value":       # the Python restatement parses "inf" like float(); C++ rejects it
        with pytest.raises(RuntimeError) as ref:
            orc.read_matrix_market(path)
        assert str(ref.value) == str(got.value)


def _random_file(rng, path, fmt, sym, rows, cols):
    lines = [f"%%MatrixMarket matrix {fmt} real {sym}", "% generated", ""]
    if fmt == "array":
        lines.append(f"{rows} {cols}")
        for j in range(cols):
            for _ in range(0 if sym == "general" else j, rows):
                lines.append(repr(float(rng.standard_normal() * 10.0 ** rng.integers(-12, 12))))
                if rng.random() < 0.05:
                    lines.append("% interleaved comment")
    else:
        nnz = int(rng.integers(0, rows * cols))
        ents = []
        for _ in range(nnz):
            i, j = int(rng.integers(1, rows + 1)), int(rng.integers(1, cols + 1))
            if sym != "general" and i < j:
                i, j = j, i
            ents.append(f"{i} {j} {float(rng.standard_normal()):.17g}")
        lines.append(f"{rows} {cols} {nnz}")
        lines += ents
    open(path, "w").write("\n".join(lines) + "\n")


@pytest.mark.parametrize("seed", range(12))
def test_random_files_bitwise_match_oracle(mm, tmp_path, seed):
    """Seeded random files (dense/sparse, general/symmetric/skew, duplicates, comments, blank
    lines): the library reader and the oracle restatement agree bit for bit, and the library's
    writer round-trips the matrix exactly."""
    s, _ = mm
    rng = np.random.default_rng(seed)
    fmt = ["array", "coordinate"][seed % 2]
    sym = ["general", "symmetric", "skew-symmetric"][(seed // 2) % 3]
    rows = int(rng.integers(1, 30))
    cols = rows if sym != "general" else int(rng.integers(1, 30))
    path = str(tmp_path / "r.mtx")
    _random_file(rng, path, fmt, sym, rows, cols)
    got, ref = s.read_matrix_market(path), orc.read_matrix_market(path)
    assert got.is_sparse() == ref.is_sparse == (fmt == "coordinate")
    assert got.transposed() == ref.transposed
    assert np.array_equal(got.to_dense(), ref.to_dense())
    if got.is_sparse():
        g, r = got.sparse(), ref.sparse
        assert np.array_equal(g.indptr, r.indptr) and np.array_equal(g.indices, r.indices)
        assert np.array_equal(g.data, r.data)
    out = str(tmp_path / "w.mtx")
    s.write_matrix_market(out, got, "seed %d" % seed)
    back = s.read_matrix_market(out)
    assert np.array_equal(back.to_dense(), got.to_dense())
    assert back.is_sparse() == got.is_sparse()


def test_from_sparse_validates_and_normalises(mm):
    s, _ = mm
    m = sp.csc_matrix(np.array([[0.0, 1.0, 0.0, 2.0], [3.0, 0.0, 0.0, 0.0]]))
    p = s.ProblemMatrix.from_sparse(m)
    assert p.transposed() and p.rows() == 4 and p.cols() == 2
    assert np.array_equal(p.to_dense(), m.toarray().T)
    bad = sp.csc_matrix(np.array([[np.nan, 1.0], [0.0, 1.0]]))
    with pytest.raises(ValueError, match="NaN/Inf"):
        s.ProblemMatrix.from_sparse(bad)
