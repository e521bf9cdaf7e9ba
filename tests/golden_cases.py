"""Decode the keys of tests/golden/sweeps.npz into (case, dtype, op, params).

Shared by the oracle pinning tests (CPU) and the CUDA parity tests (GPU), so
both run the exact list of reference outputs recorded by make_golden.py.
"""

from __future__ import annotations

import numpy as np

INPUT_SUFFIXES = ("row_ptr", "col_idx", "values", "b", "x0", "r")


def _num(tok: str, prefix: str) -> float:
    assert tok.startswith(prefix), (tok, prefix)
    return float(tok[len(prefix):])


def decode(key: str):
    parts = key.split("__")
    case = parts[0]
    if len(parts) == 2 and (parts[1] in INPUT_SUFFIXES or parts[1] == "colors"):
        return None
    if parts[1] == "prec":
        return dict(key=key, case=case, dtype="f64", op="prec", kind=parts[2], precision=parts[3])
    tag, op = parts[1], parts[2]
    rest = parts[3:]
    d = dict(key=key, case=case, dtype=tag, op=op)
    if op in ("spmv", "d", "dinv_l", "dinv_u"):
        pass
    elif op == "jr":
        d["omega"] = _num(rest[0], "w")
    elif op in ("gs", "mt"):
        d["direction"] = rest[0]
        d["omega"] = _num(rest[1], "w")
    elif op == "inner":
        d["direction"] = rest[0]
        d["n_j"] = int(_num(rest[1], "nj"))
        d["omega"] = _num(rest[2], "w")
        d["gamma"] = _num(rest[3], "g")
    elif op == "gs2":
        d["n_j"] = int(_num(rest[0], "nj"))
        d["direction"] = rest[1]
        d["form"] = rest[2]
        d["omega"] = _num(rest[3], "w")
        d["gamma"] = _num(rest[4], "g")
    elif op == "hybrid":
        d["nblocks"] = int(_num(rest[0], "P"))
        d["local"] = rest[1]
    else:
        raise KeyError(key)
    return d


def all_cases(golden: dict):
    out = []
    for k in sorted(golden):
        c = decode(k)
        if c is not None:
            out.append(c)
    return out


def inputs(golden: dict, case: str, dtype: str):
    """(row_ptr, col_idx, values, b, x0, r) cast like the reference casts (cast_matrix/cast_vector)."""
    dt = np.float32 if dtype == "f32" else np.float64
    g = golden
    vals = g[f"{case}__values"].astype(dt)
    return (g[f"{case}__row_ptr"], g[f"{case}__col_idx"], vals, g[f"{case}__b"].astype(dt),
            g[f"{case}__x0"].astype(dt), g[f"{case}__r"].astype(dt))


def regular_offsets(n: int, nblocks: int) -> np.ndarray:
    return np.linspace(0, n, nblocks + 1).round().astype(np.int64)
