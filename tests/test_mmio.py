"""MatrixMarket reader / history CSV writer (mmio.py) -- host-side, runs on CPU.

Mirrors the reference's tests/test_mmio.py, plus the reference's own outputs on
465 hand-written and fuzzed files (tests/golden/mmio.json, made by
tests/golden/make_mmio_golden.py) and the multi-threaded parser's chunk
boundaries on multi-MB files.
"""

from __future__ import annotations

import base64
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2104_01196_b200 as g2
from paper_2104_01196_b200 import MatrixMarketError, read_matrix_market, write_history_csv
from paper_2104_01196_b200.krylov import ConvergenceHistory
from paper_2104_01196_b200.sparse import from_coo

GOLDEN = Path(__file__).parent / "golden" / "mmio.json"

A2_GENERAL = [(1, 1, 2.0), (1, 2, -1.0), (2, 1, -1.0), (2, 2, 2.0)]
A2_SYMMETRIC = [(1, 1, 2.0), (2, 1, -1.0), (2, 2, 2.0)]


def write_mm(path, nrows, ncols, entries, field="real", symmetry="general"):
    lines = [f"%%MatrixMarket matrix coordinate {field} {symmetry}", f"{nrows} {ncols} {len(entries)}"]
    for e in entries:
        if field == "pattern":
            lines.append(f"{e[0]} {e[1]}")
        elif field == "integer":
            lines.append(f"{e[0]} {e[1]} {int(e[2])}")
        else:
            lines.append(f"{e[0]} {e[1]} {e[2]:.17g}")
    Path(path).write_text("\n".join(lines) + "\n")


def entries(a):
    rows = np.repeat(np.arange(a.nrows), np.diff(a.row_ptr))
    return {(int(r), int(c), float(v)) for r, c, v in zip(rows, a.col_idx, a.values)}


@pytest.fixture
def a2():
    return g2.from_dense(np.array([[2.0, -1.0], [-1.0, 2.0]]))


def _result(path, nthreads=0):
    try:
        a = read_matrix_market(path, nthreads=nthreads)
    except Exception as e:  # noqa: BLE001
        return {"error": type(e).__name__, "message": str(e)}
    return {"nrows": a.nrows, "ncols": a.ncols, "row_ptr": [int(v) for v in a.row_ptr],
            "col_idx": [int(v) for v in a.col_idx], "values": [float(v).hex() for v in a.values]}


# ------------------------------------------------ the reference's outputs on 465 files
def test_golden_reference_outputs(tmp_path):
    cases = json.loads(GOLDEN.read_text())
    assert len(cases) >= 400
    bad = []
    for c in cases:
        p = tmp_path / f"{c['name']}.mtx"
        p.write_bytes(base64.b64decode(c["data"]))
        for nt in (1, 4):
            got = _result(p, nt)
            if got != c["expect"]:
                bad.append((c["name"], nt, c["expect"], got))
    assert not bad, bad[:3]


# ------------------------------------------------ mirrors of the reference's test_mmio.py
class TestReadMatrixMarket:
    def test_general_file(self, tmp_path, a2):
        p = tmp_path / "a2.mtx"
        write_mm(p, 2, 2, A2_GENERAL)
        assert entries(read_matrix_market(p)) == entries(a2)

    def test_symmetric_expansion(self, tmp_path, a2):
        p = tmp_path / "a2s.mtx"
        write_mm(p, 2, 2, A2_SYMMETRIC, symmetry="symmetric")
        assert entries(read_matrix_market(p)) == entries(a2)

    def test_symmetric_counts(self, tmp_path):
        p = tmp_path / "s.mtx"
        write_mm(p, 3, 3, [(1, 1, 4.0), (2, 1, -1.0), (3, 1, -2.0), (3, 3, 5.0)], symmetry="symmetric")
        assert read_matrix_market(p).nnz == 2 + 2 * 2

    def test_count_mismatch_reports_eof(self, tmp_path):
        p = tmp_path / "short.mtx"
        p.write_text("%%MatrixMarket matrix coordinate real general\n3 3 3\n1 1 1.0\n2 2 2.0\n")
        with pytest.raises(MatrixMarketError, match="line 4: end of file after 2 entries"):
            read_matrix_market(p)

    def test_extra_entries_rejected(self, tmp_path):
        p = tmp_path / "long.mtx"
        p.write_text("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n2 2 2.0\n")
        with pytest.raises(MatrixMarketError, match="line 4"):
            read_matrix_market(p)

    def test_bad_banner(self, tmp_path):
        p = tmp_path / "bad.mtx"
        p.write_text("%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 1.0\n")
        with pytest.raises(MatrixMarketError, match="line 1"):
            read_matrix_market(p)

    def test_complex_field_rejected(self, tmp_path):
        p = tmp_path / "cplx.mtx"
        p.write_text("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1.0 0.0\n")
        with pytest.raises(MatrixMarketError, match="complex"):
            read_matrix_market(p)

    def test_hermitian_rejected(self, tmp_path):
        p = tmp_path / "herm.mtx"
        p.write_text("%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1.0\n")
        with pytest.raises(MatrixMarketError, match="hermitian"):
            read_matrix_market(p)

    def test_index_out_of_bounds_has_line_number(self, tmp_path):
        p = tmp_path / "oob.mtx"
        p.write_text("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n3 1 1.0\n")
        with pytest.raises(MatrixMarketError, match=r"line 4: index \(3, 1\) outside declared bounds 2x2"):
            read_matrix_market(p)

    def test_pattern_gets_unit_values(self, tmp_path):
        p = tmp_path / "pat.mtx"
        write_mm(p, 2, 2, [(1, 1), (2, 2), (2, 1)], field="pattern")
        assert np.all(read_matrix_market(p).values == 1.0)

    def test_integer_parsed_as_real(self, tmp_path):
        p = tmp_path / "int.mtx"
        write_mm(p, 2, 2, [(1, 1, 3), (2, 2, 7)], field="integer")
        got = read_matrix_market(p)
        assert got.values.dtype == np.float64
        assert np.array_equal(np.diag(got.to_dense()), [3.0, 7.0])

    def test_duplicates_summed(self, tmp_path):
        p = tmp_path / "dup.mtx"
        write_mm(p, 2, 2, [(1, 1, 1.0), (1, 1, 2.5), (2, 2, 1.0)])
        assert read_matrix_market(p).to_dense()[0, 0] == 3.5

    def test_comments_and_blank_lines_skipped(self, tmp_path):
        p = tmp_path / "com.mtx"
        p.write_text("%%MatrixMarket matrix coordinate real general\n% a comment\n\n2 2 2\n% another\n"
                     "1 1 1.5\n\n2 2 2.5\n")
        assert np.array_equal(np.diag(read_matrix_market(p).to_dense()), [1.5, 2.5])

    def test_round_trip_idempotent(self, tmp_path):
        rng = np.random.default_rng(4)
        ents = [(int(i) + 1, int(j) + 1, float(v)) for i, j, v in
                zip(rng.integers(0, 8, 30), rng.integers(0, 8, 30), rng.uniform(-2, 2, 30))]
        p1 = tmp_path / "r1.mtx"
        write_mm(p1, 8, 8, ents)
        a1 = read_matrix_market(p1)
        rows = np.repeat(np.arange(8), np.diff(a1.row_ptr))
        p2 = tmp_path / "r2.mtx"
        write_mm(p2, 8, 8, [(int(r) + 1, int(c) + 1, float(v)) for r, c, v in zip(rows, a1.col_idx, a1.values)])
        assert entries(a1) == entries(read_matrix_market(p2))

    def test_trefethen_20_structure(self, tmp_path):
        """SuiteSparse JGD_Trefethen/Trefethen_20 (the reference's fixture), regenerated from its
        definition: primes on the diagonal, 1 where |i-j| is a power of two; symmetric integer."""
        primes = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53, 59, 61, 67, 71]
        lower = [(i, i, primes[i - 1]) for i in range(1, 21)]
        lower += [(i, j, 1) for i in range(1, 21) for j in range(1, i) if (i - j) & (i - j - 1) == 0]
        p = tmp_path / "trefethen_20.mtx"
        write_mm(p, 20, 20, lower, field="integer", symmetry="symmetric")
        a = read_matrix_market(p)
        assert a.nrows == a.ncols == 20
        assert a.nnz == 158  # 89 stored, off-diagonals mirrored
        d = a.to_dense()
        assert np.array_equal(d, d.T)
        assert np.array_equal(np.diag(d), primes)

    def test_reference_fixture_if_present(self):
        path = Path("/root/reference/pkg/tests/data/trefethen_20.mtx")
        if not path.exists():
            pytest.skip("reference checkout not present")
        a = read_matrix_market(path)
        assert a.nnz == 158 and np.array_equal(np.diag(a.to_dense())[:4], [2, 3, 5, 7])


# ------------------------------------------------ the threaded parser on multi-MB inputs
def _big_file(path, rng, n=50_000, m=400_000, breaks=(b"\n", b"\r\n", b"\r")):
    r = rng.integers(1, n + 1, m)
    c = rng.integers(1, n + 1, m)
    v = rng.standard_normal(m)
    br = [breaks[k] for k in rng.integers(0, len(breaks), m)]
    body = b"".join(f"{a} {b} {x:.17g}".encode() + e for a, b, x, e in zip(r, c, v, br))
    head = f"%%MatrixMarket matrix coordinate real general\n% big\n{n} {n} {m}\n".encode()
    Path(path).write_bytes(head + body)
    return n, r - 1, c - 1, v, head, body


def test_threaded_parse_matches_single_thread_and_from_coo(tmp_path):
    rng = np.random.default_rng(7)
    p = tmp_path / "big.mtx"
    n, r, c, v, _, _ = _big_file(p, rng)
    assert p.stat().st_size > 8 << 20  # several 1 MB thread ranges
    a1 = read_matrix_market(p, nthreads=1)
    a8 = read_matrix_market(p, nthreads=8)
    want = from_coo(n, n, r, c, v)
    for a in (a1, a8):
        assert np.array_equal(a.row_ptr, want.row_ptr)
        assert np.array_equal(a.col_idx, want.col_idx)
        assert np.array_equal(a.values.view(np.int64), want.values.view(np.int64))


@pytest.mark.parametrize("where", [0.25, 0.5, 0.999])
def test_threaded_parse_reports_first_bad_line(tmp_path, where):
    rng = np.random.default_rng(11)
    p = tmp_path / "big.mtx"
    n, r, c, v, head, body = _big_file(p, rng, breaks=(b"\n",))
    lines = body.split(b"\n")
    k = int(where * (len(lines) - 2))
    lines[k] = b"1 1 1.0.0"
    lines[k + 7] = b"1 1"  # a later error must not win
    p.write_bytes(head + b"\n".join(lines))
    lineno = 3 + k + 1
    for nt in (1, 8):
        with pytest.raises(MatrixMarketError, match=rf"^line {lineno}: cannot parse entry '1 1 1.0.0'$"):
            read_matrix_market(p, nthreads=nt)


def test_from_coo_order_matches_lexsort():
    rng = np.random.default_rng(3)
    for _ in range(30):
        n = int(rng.integers(1, 60))
        m = int(rng.integers(0, 500))
        r, c, v = rng.integers(0, n, m), rng.integers(0, n, m), rng.standard_normal(m)
        a = from_coo(n, n, r, c, v)
        o = np.lexsort((c, r))
        rr, cc, vv = r[o], c[o], v[o]
        if m:
            f = np.ones(m, bool)
            f[1:] = (rr[1:] != rr[:-1]) | (cc[1:] != cc[:-1])
            s = np.flatnonzero(f)
            vv, rr, cc = np.add.reduceat(vv, s), rr[s], cc[s]
        assert np.array_equal(a.col_idx, cc)
        assert np.array_equal(a.values.view(np.int64), vv.view(np.int64))
        assert np.array_equal(a.row_ptr, np.concatenate([[0], np.cumsum(np.bincount(rr, minlength=n))]))


# ------------------------------------------------ write_history_csv (mmio.py:109-120)
class TestHistoryCsv:
    def test_single_entry(self, tmp_path):
        p = tmp_path / "h.csv"
        write_history_csv(ConvergenceHistory(np.array([1.0]), False), {"solver": "cg", "n": 5}, p)
        lines = p.read_text().splitlines()
        assert lines[0].startswith("# solver=cg")
        assert lines[1] == "iter,rel_res"
        assert lines[2] == "0,1"
        assert len(lines) == 3

    def test_round_trip_bitwise(self, tmp_path):
        values = np.array([1.0, 1.0 / 3.0, 2.3e-11, 7.123456789012345e-101])
        p = tmp_path / "h.csv"
        write_history_csv(ConvergenceHistory(values, True), {"n": 4}, p)
        parsed = [float(line.split(",")[1]) for line in p.read_text().splitlines()[2:]]
        assert np.array_equal(np.array(parsed), values)

    def test_unwritable_path(self, tmp_path):
        with pytest.raises(OSError):
            write_history_csv(ConvergenceHistory(np.array([1.0]), False), {}, tmp_path / "missing" / "h.csv")
