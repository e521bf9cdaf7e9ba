"""Kernel microbenchmarks on one B200 (CUDA events, warm, inputs >> L2).

    python profiles/microbench.py [--n 16777216] [--which cgs,precond,spmv,sweep]

Prints one JSON line per (kernel, k) with ms and algorithmic GB/s; used to
choose between kernel variants before a bench run.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2104_01196_b200 as g2  # noqa: E402
from paper_2104_01196_b200 import _native  # noqa: E402


def p(t):
    return C.c_void_p(t.data_ptr())


def timeit(fn, reps=10):
    st = fn()
    if isinstance(st, int):
        _native.check(st, "microbench")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=256)
    ap.add_argument("--which", default="cgs,precond,spmv,sweep")
    ap.add_argument("--ks", default="1,8,31,61")
    args = ap.parse_args()
    lib = _native.load()
    nx = args.nx
    n = nx ** 3
    V8 = 8 * n
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    which = args.which.split(",")
    ks = [int(k) for k in args.ks.split(",")]
    if "cgs" in which:
        kmax = max(ks)
        V = torch.randn(kmax + 1, n, dtype=torch.float64, device="cuda")
        w = torch.randn(n, dtype=torch.float64, device="cuda")
        h = torch.randn(kmax + 1, dtype=torch.float64, device="cuda") * 1e-3
        h2 = torch.empty_like(h)
        nrm = torch.empty(1, dtype=torch.float64, device="cuda")
        work = torch.zeros(int(lib.rs_reduce_work_doubles(kmax + 2)), dtype=torch.float64, device="cuda")
        for k in ks:
            res = {
                "gemv_t": (timeit(lambda: lib.rs_gemv_t(p(V), n, k, n, p(w), p(h2), None, p(work), st)), (k + 1) * V8),
                "gemv_n_update": (timeit(lambda: lib.rs_gemv_n_update(p(V), n, k, n, p(h), p(w), None, p(work), st)),
                                  (k + 2) * V8),
                "cgs_dots": (timeit(lambda: lib.rs_cgs_pass(p(V), n, k, n, None, p(w), p(h2), None, None, p(work), st)),
                             (k + 1) * V8),
                "cgs_update_dots": (timeit(lambda: lib.rs_cgs_pass(p(V), n, k, n, p(h), p(w), p(h2), None, None,
                                                                   p(work), st)), (k + 2) * V8),
                "cgs_update_norm": (timeit(lambda: lib.rs_cgs_pass(p(V), n, k, n, p(h), p(w), None, p(nrm), None,
                                                                   p(work), st)), (k + 2) * V8),
            }
            for name, (ms, by) in res.items():
                print(json.dumps({"kernel": name, "k": k, "ms": round(ms, 4), "gbs": round(by / ms / 1e6, 1)}),
                      flush=True)
        del V
    if "precond" in which or "spmv" in which or "sweep" in which:
        a = g2.laplace3d(nx, device="cuda")
        ML = 12 * a.nnz_l + 4 * (n + 1)
        MU = 12 * a.nnz_u + 4 * (n + 1)
        r = g2.random_rhs(n, 0, device="cuda")
        z = torch.empty_like(r)
        if "precond" in which:
            for nj in (0, 1, 2):
                pc = g2.Preconditioner(a, "gs2", g2.RelaxConfig(1, 1, nj))
                by = 3 * V8 if nj == 0 else (ML + 3 * V8 if nj == 1 else 2 * ML + 7 * V8)
                ms = timeit(lambda: pc.apply_into(r, z))
                print(json.dumps({"kernel": f"precond_gs2_nj{nj}", "ms": round(ms, 4), "gbs": round(by / ms / 1e6, 1)}),
                      flush=True)
            for nj in (1, 2):
                pc = g2.Preconditioner(a, "gs2", g2.RelaxConfig(1, 1, nj), precision="single_inside_double")
                by = nj * (4 * a.nnz_l * 2 + 4 * (n + 1)) + 8 * n + 4 * n + 8 * n
                ms = timeit(lambda: pc.apply_into(r, z))
                print(json.dumps({"kernel": f"precond_gs2_nj{nj}_f32", "ms": round(ms, 4),
                                  "gbs": round(by / ms / 1e6, 1)}), flush=True)
        if "sweep" in which:
            from paper_2104_01196_b200 import _native as NN
            b = g2.random_rhs(n, 0, device="cuda")
            x0 = g2.random_rhs(n, 1, device="cuda")
            x1 = torch.empty_like(x0)
            for nj in (1, 2, 3):
                cfg = NN.RelaxCfg.of(g2.RelaxConfig(1, 1, nj))
                model = ML + MU + 4 * V8 + (ML + 3 * V8 if nj == 1 else (ML + 2 * V8) + (nj - 2) * (ML + 3 * V8) + (ML + 4 * V8))
                ms = timeit(lambda: lib.rs_gs2_sweep(a.handle, p(b), p(x0), p(x1), C.byref(cfg), st))
                print(json.dumps({"kernel": f"gs2_sweep_oop_nj{nj}", "ms": round(ms, 4),
                                  "model_gbs": round(model / ms / 1e6, 1)}), flush=True)
                ms = timeit(lambda: lib.rs_gs2_apply(a.handle, p(b), p(x0), C.byref(cfg), st))
                print(json.dumps({"kernel": f"gs2_apply_inplace_nj{nj}", "ms": round(ms, 4),
                                  "model_gbs": round(model / ms / 1e6, 1)}), flush=True)
        if "spmv" in which:
            y = torch.empty_like(r)
            ms = timeit(lambda: lib.rs_spmv(a.handle, p(r), None, None, p(y), st))
            print(json.dumps({"kernel": "spmv", "ms": round(ms, 4), "gbs": round((ML + MU + 3 * V8) / ms / 1e6, 1)}),
                  flush=True)
        # copy roofline reference on this GPU
        big = torch.empty(2 * n, dtype=torch.float64, device="cuda")
        big2 = torch.empty_like(big)
        ms = timeit(lambda: big2.copy_(big))
        print(json.dumps({"kernel": "torch_copy", "ms": round(ms, 4), "gbs": round(2 * 16 * n / ms / 1e6, 1)}))


if __name__ == "__main__":
    main()
