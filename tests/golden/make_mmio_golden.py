"""Generate tests/golden/mmio.json by running the REFERENCE MatrixMarket reader.

Test infrastructure: imports the reference package (`relaxsolve`,
/root/reference/pkg/src) in THIS container, feeds it a deterministic set of
MatrixMarket files -- hand-written edge cases plus seeded byte-level mutations
of valid files -- and records, per file, either the exact exception message
(`MatrixMarketError` / other) or the resulting CSR (values as float.hex()).
The fixture travels with the repo; the reference does not.

    python tests/golden/make_mmio_golden.py
"""

from __future__ import annotations

import base64
import json
import random
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")

import relaxsolve as rs  # noqa: E402

HERE = Path(__file__).parent

HDR = "%%MatrixMarket matrix coordinate {field} {sym}\n"


def valid_files():
    """(name, bytes) of well-formed files that exercise the grammar."""
    out = []
    r = "%%MatrixMarket matrix coordinate real general\n"
    out.append(("general", (r + "3 3 4\n1 1 2.0\n2 2 -1.5e-3\n3 1 7\n3 3 .5\n").encode()))
    out.append(("crlf", (r + "2 2 2\r\n1 1 1.25\r\n2 2 2.5\r\n").replace("\n", "\r\n").encode()))
    out.append(("cr_only", (r.replace("\n", "\r") + "2 2 2\r1 1 1.25\r2 2 2.5\r").encode()))
    out.append(("mixed_breaks", (r + "2 2 3\r\n1 1 1\r2 2 2\n\r\n1 2 3").encode()))
    out.append(("no_final_break", (r + "2 2 2\n1 1 1\n2 2 2").encode()))
    out.append(("tabs_ff", (r + "2\t2 2\n\t1\x0c1\t1e0 \n 2 2\x0b2\x1c\n").encode()))
    out.append(("comments_blank", (r + "% c\n\n  \n3 3 2\n% mid\n\n1 1 1\n   % indented\n3 3 3\n\n").encode()))
    out.append(("underscores", (r + "2 2 3\n1_0 1 1_000.5\n1 1 1e1_0\n2 2 0.0_1\n").replace("2 2 3", "10 10 3").encode()))
    out.append(("signs_zeros", (r + "3 3 3\n+1 001 -0.0\n0002 +2 +1.5E+2\n3 3 -.25e-1\n").encode()))
    out.append(("specials", (r + "3 3 5\n1 1 inf\n2 2 -Infinity\n3 3 nan\n1 2 iNF\n2 1 -NaN\n").encode()))
    out.append(("extremes", (r + "3 3 4\n1 1 1e400\n2 2 4.9e-324\n3 3 2.4703282292062328e-324\n"
                             "1 3 0.1000000000000000055511151231257827021181583404541015625\n").encode()))
    out.append(("long_digits", (r + "1 1 1\n1 1 " + "9" * 80 + "." + "1" * 80 + "e-60\n").encode()))
    out.append(("dup_sum", (r + "2 2 5\n1 1 0.1\n1 1 0.2\n2 2 1\n1 1 0.3\n2 2 1e-17\n").encode()))
    out.append(("pattern", (HDR.format(field="pattern", sym="general") + "3 3 3\n1 1\n3 2\n2 3\n").encode()))
    out.append(("integer", (HDR.format(field="integer", sym="general") + "2 2 2\n1 1 3\n2 2 -7\n").encode()))
    out.append(("integer_float", (HDR.format(field="integer", sym="general") + "2 2 1\n1 1 3.5\n").encode()))
    out.append(("symmetric", (HDR.format(field="real", sym="symmetric")
                              + "3 3 4\n1 1 4\n2 1 -1\n3 1 -2\n3 3 5\n").encode()))
    out.append(("sym_pattern", (HDR.format(field="pattern", sym="symmetric") + "3 3 3\n1 1\n3 1\n2 1\n").encode()))
    out.append(("upper_banner", b"%%MatrixMarket MATRIX Coordinate REAL General\n2 2 1\n2 2 1\n"))
    out.append(("empty_matrix", (r + "0 0 0\n").encode()))
    out.append(("zero_entries", (r + "4 4 0\n% nothing\n").encode()))
    out.append(("rect", (r + "2 4 3\n1 4 1\n2 1 2\n2 3 3\n").encode()))
    out.append(("high_bytes_comment", (r + "%\xe9\xff comment\n1 1 1\n1 1 1\n").encode("latin-1")))
    return out


def invalid_files():
    r = "%%MatrixMarket matrix coordinate real general\n"
    out = [
        ("empty", b""),
        ("only_break", b"\n"),
        ("bad_banner", b"%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 1.0\n"),
        ("banner_4_parts", b"%%MatrixMarket matrix coordinate real\n1 1 1\n1 1 1\n"),
        ("banner_quote", b"%%MatrixMarket it's bad\n"),
        ("complex", b"%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1.0 0.0\n"),
        ("hermitian", b"%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1.0\n"),
        ("array", b"%%MatrixMarket matrix array real general\n1 1\n1.0\n"),
        ("vector", b"%%MatrixMarket vector coordinate real general\n1 1 1\n1 1 1\n"),
        ("missing_size", (r + "% only comments\n\n").encode()),
        ("missing_size_nolines", r.encode()),
        ("size_2", (r + "3 3\n").encode()),
        ("size_float", (r + "3 3 1.0\n1 1 1\n").encode()),
        ("size_negative", (r + "3 -3 1\n1 1 1\n").encode()),
        ("short", (r + "3 3 3\n1 1 1.0\n2 2 2.0\n").encode()),
        ("short_no_break", (r + "3 3 3\n1 1 1.0\n2 2 2.0").encode()),
        ("short_trailing_comment", (r + "3 3 3\n1 1 1.0\n% end\n\n").encode()),
        ("long", (r + "2 2 1\n1 1 1.0\n2 2 2.0\n").encode()),
        ("long_after_blank", (r + "2 2 1\n1 1 1.0\n\n% c\n2 2 2.0\n").encode()),
        ("oob_row", (r + "2 2 2\n1 1 1.0\n3 1 1.0\n").encode()),
        ("oob_zero", (r + "2 2 1\n0 1 1.0\n").encode()),
        ("oob_neg", (r + "2 2 1\n-1 1 1.0\n").encode()),
        ("oob_huge", (r + "2 2 1\n1 99999999999999999999999 1.0\n").encode()),
        ("fields_2", (r + "2 2 1\n1 1\n").encode()),
        ("fields_4", (r + "2 2 1\n1 1 1 1\n").encode()),
        ("pattern_3", (HDR.format(field="pattern", sym="general") + "2 2 1\n1 1 1\n").encode()),
        ("float_index", (r + "2 2 1\n1.0 1 1\n").encode()),
        ("hex_value", (r + "2 2 1\n1 1 0x10\n").encode()),
        ("hexfloat_value", (r + "2 2 1\n1 1 0x1p3\n").encode()),
        ("double_underscore", (r + "2 2 1\n1 1 1__0\n").encode()),
        ("lead_underscore", (r + "2 2 1\n_1 1 1\n").encode()),
        ("trail_underscore", (r + "2 2 1\n1 1 1_\n").encode()),
        ("underscore_dot", (r + "2 2 1\n1 1 1_.5\n").encode()),
        ("bare_e", (r + "2 2 1\n1 1 1e\n").encode()),
        ("bare_dot", (r + "2 2 1\n1 1 .\n").encode()),
        ("nan_payload", (r + "2 2 1\n1 1 nan(1)\n").encode()),
        ("infinit", (r + "2 2 1\n1 1 infinit\n").encode()),
        ("double_sign", (r + "2 2 1\n1 1 --1\n").encode()),
        ("nul_byte", (r + "2 2 1\n1 1 1\x00\n").encode()),
        ("high_byte_value", (r + "2 2 1\n1 1 1\xe9\n").encode("latin-1")),
        ("nbsp_sep", (r + "2 2 1\n1\xa01 1\n").encode("latin-1")),
        ("first_error_wins", (r + "3 3 3\n1 1 x\n9 9 1\n1 1 1\n1 1 1\n").encode()),
    ]
    return out


def mutate(rng: random.Random, data: bytes) -> bytes:
    b = bytearray(data)
    for _ in range(rng.randint(1, 3)):
        op = rng.randrange(6)
        if not b:
            break
        i = rng.randrange(len(b))
        if op == 0:
            b[i] = rng.choice(b" \t\n\r0123456789.-+eE_%x\x00\x85\xff\x0c\x1c")
        elif op == 1:
            del b[i]
        elif op == 2:
            b.insert(i, rng.choice(b" \n\r9.e_-%"))
        elif op == 3:  # duplicate a line
            s = data.split(b"\n")
            k = rng.randrange(len(s))
            s.insert(k, s[k])
            b = bytearray(b"\n".join(s))
        elif op == 4:  # delete a line
            s = bytes(b).split(b"\n")
            if len(s) > 2:
                del s[rng.randrange(1, len(s))]
            b = bytearray(b"\n".join(s))
        else:
            b[i:i] = rng.choice([b"1e999", b"_", b"  ", b"\r\n", b"inf", b"007", b"+", b"%"])
    return bytes(b)


def seed_file(rng: random.Random) -> bytes:
    n = rng.randint(1, 6)
    field = rng.choice(["real", "integer", "pattern"])
    sym = rng.choice(["general", "symmetric"])
    ents = []
    for _ in range(rng.randint(0, 8)):
        i, j = rng.randint(1, n), rng.randint(1, n)
        if sym == "symmetric" and j > i:
            i, j = j, i
        if field == "pattern":
            ents.append(f"{i} {j}")
        elif field == "integer":
            ents.append(f"{i} {j} {rng.randint(-9, 9)}")
        else:
            ents.append(f"{i} {j} {rng.uniform(-2, 2):.17g}")
    body = "\n".join(ents)
    return (HDR.format(field=field, sym=sym) + f"{n} {n} {len(ents)}\n" + body + ("\n" if ents else "")).encode()


def run_reference(data: bytes):
    with tempfile.NamedTemporaryFile(suffix=".mtx", delete=False) as fh:
        fh.write(data)
        path = fh.name
    try:
        a = rs.read_matrix_market(path)
    except Exception as e:  # noqa: BLE001 -- the type and message are the fixture
        return {"error": type(e).__name__, "message": str(e)}
    finally:
        Path(path).unlink()
    return {
        "nrows": a.nrows, "ncols": a.ncols,
        "row_ptr": [int(v) for v in a.row_ptr], "col_idx": [int(v) for v in a.col_idx],
        "values": [float(v).hex() for v in a.values],
    }


def main():
    rng = random.Random(2104_01196)
    cases = valid_files() + invalid_files()
    for k in range(400):
        base = seed_file(rng) if k % 2 else rng.choice(valid_files())[1]
        cases.append((f"fuzz{k:03d}", mutate(rng, base)))
    out = []
    for name, data in cases:
        out.append({"name": name, "data": base64.b64encode(data).decode(), "expect": run_reference(data)})
    (HERE / "mmio.json").write_text(json.dumps(out, indent=0))
    nerr = sum("error" in c["expect"] for c in out)
    print(f"{len(out)} cases ({nerr} errors) -> {HERE / 'mmio.json'}")


if __name__ == "__main__":
    main()
