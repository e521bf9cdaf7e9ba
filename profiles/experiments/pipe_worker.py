"""Run every GS2 sweep flavour on a few matrices and save the iterates (tests/test_pipe.py).

The window-pipelined one-launch sweep (relax.cu k_gs2_pipe) is chosen by environment
variables read once per process (RS_PIPE=0 disables it, RS_PIPE_WS sets the minimum log2
window), so the test runs this script in subprocesses and compares their outputs bitwise.

    python tests/pipe_worker.py OUT.npz
"""

from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import paper_2104_01196_b200 as g2  # noqa: E402
from paper_2104_01196_b200 import _native  # noqa: E402


def banded_random(n, bw, seed, dtype):
    """Structurally non-symmetric random matrix, |i - j| <= bw, dominant diagonal."""
    rng = np.random.default_rng(seed)
    rows, cols, vals = [np.arange(n)], [np.arange(n)], [np.full(n, 8.0)]
    for _ in range(4):
        i = rng.integers(0, n, size=n)
        j = np.clip(i + rng.integers(-bw, bw + 1, size=n), 0, n - 1)
        rows.append(i)
        cols.append(j)
        vals.append(rng.uniform(-1, 1, size=n))
    r, c, v = (np.concatenate(t) for t in (rows, cols, vals))
    return g2.from_coo(n, n, r, c, v.astype(dtype), dtype=dtype)


def matrices(dtype):
    mats = [("lap3d_20", g2.laplace3d(20)), ("lap3d_17x13x9", g2.laplace3d(17, 13, 9)),
            ("convdiff_16", g2.convdiff3d(16)), ("elast_5", g2.elasticity3d(5)),
            ("band_3000", banded_random(3000, 150, 7, np.float64))]
    for name, a in mats:
        yield name, (g2.cast_matrix(a, "single") if dtype == np.float32 else a)


def main():
    out = {}
    lib = _native.load()
    for dtype in (np.float64, np.float32):
        tag = "f64" if dtype == np.float64 else "f32"
        for name, a in matrices(dtype):
            n = a.nrows
            b = g2.random_rhs(n, 0).astype(dtype)
            x0 = g2.random_rhs(n, 1).astype(dtype)
            for n_j in (1, 2, 3, 5):
                for direction in ("forward", "backward", "symmetric"):
                    for form in ("non_compact", "compact"):
                        for om, gm in ((1.0, 1.0), (1.3, 0.8)):
                            cfg = g2.RelaxConfig(2, 1, n_j, direction, form, om, gm)
                            s = g2.extract_splitting(a, omega=om, gamma=gm)
                            x = x0.copy()
                            l0 = lib.rs_launch_count()
                            g2.gs2_apply(a, s, b, x, cfg)
                            key = f"{tag}/{name}/sweep/{n_j}/{direction}/{form}/{om}/{gm}"
                            out[key] = x
                            out["launches:" + key] = np.array(lib.rs_launch_count() - l0)
                            if form == "compact":
                                continue
                            if tag != "f64":  # Preconditioner needs a double-precision matrix
                                continue
                            for prec in ("same", "single_inside_double"):
                                m = g2.Preconditioner(a, "gs2", g2.RelaxConfig(1, 1, n_j, direction, form, om, gm),
                                                      precision=prec)
                                out[f"{tag}/{name}/prec/{n_j}/{direction}/{om}/{gm}/{prec}"] = m.apply(
                                    b.astype(np.float64))
    np.savez(sys.argv[1], **out)
    print("PIPE_WORKER_OK", len(out))


if __name__ == "__main__":
    main()
