"""The reference-side bindings of INTEGRATION.md, executed.

* §C: the ctypes binding of the numba kernel ABI (csr_matvec, gs_ordered_sweep; _kernels.py:15-39)
  is taken verbatim from INTEGRATION.md, pointed at the built library, and driven exactly the way
  the reference drives the numba kernels (int64 CSR arrays, the `order` array of relax.py:160-190 /
  coloring.py:66-88, omega and 1 - omega pre-cast to the dtype as relax.py:171-174 does); every
  golden SpMV / sequential-GS / multicolour-GS output is reproduced bit for bit.
* §B: the GPU Preconditioner inside a reference-style MGS GMRES loop (krylov.py:162-250, restated
  below as test infrastructure: numpy on the host, `m.apply` on numpy arrays): config 1's counts.
"""

import re
from pathlib import Path

import numpy as np
import pytest

import paper_2104_01196_b200 as g2
from golden_cases import all_cases, inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = Path(__file__).resolve().parent.parent


def _section_code(title: str) -> str:
    text = (ROOT / "INTEGRATION.md").read_text()
    sec = text[text.index(title):]
    m = re.search(r"```python\n(.*?)```", sec, re.S)
    return m.group(1)


@pytest.fixture(scope="module")
def shim():
    from paper_2104_01196_b200 import build

    code = _section_code("## C. Binding the C ABI from the reference")
    code = code.replace('ctypes.CDLL("libgs2b200.so")', f"ctypes.CDLL({str(build.build())!r})")
    ns = {}
    exec(compile(code, "INTEGRATION.md#C", "exec"), ns)  # noqa: S102 -- the documented binding itself
    return ns


def _colour_classes(colors):
    return [np.flatnonzero(colors == c).astype(np.int64) for c in range(int(colors.max()) + 1)]


def test_numba_abi_shim_bitwise_on_golden_fixtures(shim, sweeps_golden):
    csr_matvec, gs_ordered_sweep = shim["csr_matvec"], shim["gs_ordered_sweep"]
    done = {"spmv": 0, "gs": 0, "mt": 0}
    for c in all_cases(sweeps_golden):
        if c["op"] not in done:
            continue
        rp, ci, v, b, x0, _ = inputs(sweeps_golden, c["case"], c["dtype"])
        dt = v.dtype.type
        want = sweeps_golden[c["key"]]
        n = len(rp) - 1
        if c["op"] == "spmv":
            out = np.empty(n, dtype=v.dtype)
            csr_matvec(rp, ci, v, x0, out)
        else:
            w, w1 = dt(c["omega"]), dt(1.0 - c["omega"])  # relax.py:171-174
            diag = np.array([v[k] for i in range(n) for k in range(rp[i], rp[i + 1]) if ci[k] == i], dtype=v.dtype)
            dirs = ("forward", "backward") if c["direction"] == "symmetric" else (c["direction"],)
            out = x0.copy()
            for d in dirs:
                if c["op"] == "gs":
                    order = np.arange(n, dtype=np.int64)
                    if d == "backward":
                        order = order[::-1].copy()
                else:
                    groups = _colour_classes(sweeps_golden[f"{c['case']}__colors"])
                    order = np.concatenate(groups if d == "forward" else groups[::-1])
                gs_ordered_sweep(rp, ci, v, diag, b, out, order, w, w1)
        assert np.array_equal(out, want), c["key"]
        done[c["op"]] += 1
    assert min(done.values()) > 0, done


def _reference_style_gmres(a_matvec, b, apply_m, restart, tol=1e-9, maxit=10000):
    """krylov.py:162-250 restated (test infrastructure): MGS Arnoldi, Givens, right preconditioning."""
    n = b.shape[0]
    x = np.zeros(n)
    bnorm = np.linalg.norm(b)
    r = b - a_matvec(x)
    hist = [np.linalg.norm(r) / bnorm]
    total, converged = 0, False
    while total < maxit and not converged:
        beta = np.linalg.norm(r)
        v = np.empty((restart + 1, n))
        h = np.zeros((restart + 1, restart))
        cs, sn, g = np.zeros(restart), np.zeros(restart), np.zeros(restart + 1)
        v[0] = r / beta
        g[0] = beta
        j = -1
        while j + 1 < restart and total < maxit:
            j += 1
            total += 1
            w = a_matvec(apply_m(v[j]))
            for i in range(j + 1):
                h[i, j] = v[i] @ w
                w -= h[i, j] * v[i]
            h[j + 1, j] = np.linalg.norm(w)
            v[j + 1] = w / h[j + 1, j]
            for i in range(j):
                hi = cs[i] * h[i, j] + sn[i] * h[i + 1, j]
                h[i + 1, j] = -sn[i] * h[i, j] + cs[i] * h[i + 1, j]
                h[i, j] = hi
            denom = np.hypot(h[j, j], h[j + 1, j])
            cs[j], sn[j] = h[j, j] / denom, h[j + 1, j] / denom
            h[j, j], h[j + 1, j] = denom, 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            est = abs(g[j + 1]) / bnorm
            hist.append(est)
            if est <= tol:
                break
        y = np.zeros(j + 1)
        for i in range(j, -1, -1):
            y[i] = (g[i] - h[i, i + 1:j + 1] @ y[i + 1:j + 1]) / h[i, i]
        x += apply_m(v[: j + 1].T @ y)
        r = b - a_matvec(x)
        hist[-1] = np.linalg.norm(r) / bnorm
        converged = hist[-1] <= tol
    return x, hist, converged


@pytest.mark.parametrize("kind,cfg,want", [("gs2", (2, 1, 1), 563), ("gs_seq", (2, 1, 0), 471)])
def test_gpu_preconditioner_in_reference_gmres_seam(shim, kind, cfg, want):
    """the GPU Preconditioner's numpy-in / numpy-out apply inside the reference's
    MGS loop; the SpMV is the §C shim, so the whole loop runs on the reference seams."""
    a = g2.laplace2d(128)
    b = g2.random_rhs(a.nrows, 0)
    m = g2.Preconditioner(a, kind, g2.RelaxConfig(*cfg))
    rp, ci, v = a.row_ptr, a.col_idx, a.values

    def matvec(x):
        out = np.empty(a.nrows)
        shim["csr_matvec"](rp, ci, v, x, out)
        return out

    _, hist, conv = _reference_style_gmres(matvec, b, m.apply, restart=30)
    assert conv and len(hist) - 1 == want
