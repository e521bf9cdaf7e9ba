#!/usr/bin/env python
"""bench.py -- GS2-preconditioned GMRES(60) on B200 (BASELINE.json metric / configs).

One step = one full GMRES(60) restart cycle (60 Arnoldi iterations, each one zero-start
GS2(1,1,1) preconditioner application + one SpMV + DCGS2 orthogonalisation, then the cycle-end
update and true residual) on the synthetic 3D 7-point Laplace problem, b = random_rhs(n, 0):

* N = 1: config C2, laplace3d 256^3 (16.7 M rows) on one B200.
* N > 1: config C5, laplace3d 512^3 row-partitioned into N z-slabs (one rank per GPU; hybrid
  block-Jacobi GS2 preconditioner; halo exchange and the Gram-Schmidt allreduces over NVLink peer
  memory, the allreduces fused into the CGS kernels -- ``--comm nccl`` for the NCCL baseline).
  ``python bench.py --gpus N`` re-executes itself under ``torch.distributed.run`` with N ranks
  when it is not already running under a launcher (WORLD_SIZE unset); rank 0 prints the line.

``value`` (GB/s, higher is better) = W / t: W = the algorithmic HBM bytes of the kernel sequence
the B200 path launches for the step's work (split-CSR int32 + fp64, each operand once per pass,
fused passes counted once; summed over ranks), t = device time of the step (max over ranks).
For our arm W is exactly the bytes the kernels must move, so value / the measured copy peak is
the whole-cycle roofline fraction.  The reference arm (``--impl reference``) times the
reference's CPU algorithm (the C oracle port, all host threads) on Arnoldi iterations sampled
across the same 60-step cycle (stratified j) and divides the SAME W of those iterations by its
time, so the driver's ratio of the two values is the time ratio on identical work; the oracle's
own byte count is reported beside it.  The SURVEY §8(d) model bytes (unfused CGS2) stay as
``config.model_bytes_per_step`` / ``model_gbs``.

Extra keys of the N = 1 line: ``sweeps`` (the metric's GS2 sweep GB/s and the paper's
same-device baselines: JR, level-scheduled GS, multicolour GS, n_j = 0..3), ``tts`` (time to
solution), ``c5_one_gpu`` (the 512^3 cycle on one GPU: the strong-scaling reference of the
N > 1 lines), ``configs`` (C1, C3, C4 and the stand-alone smoother), ``setup`` (matrix build /
split, level-set analysis, colouring), ``cpu_baseline`` (the oracle on one core).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "GMRES+GS2 time-to-solution & GS2 sweep GB/s vs HBM peak at 1/2/4/8 B200"


# ---------------------------------------------------------------- byte model
class Model:
    """Algorithmic bytes of each kernel of the path (each operand once per pass).

    Matrix bytes per triangle: split-CSR (int32 idx, fp64 values, the SURVEY §8(d) figure) or, for a
    stencil-encoded triangle (rs_mat_layout stencil_k > 0: constant-coefficient stencils such as
    laplace3d / convdiff3d), the 32-byte lane-mask row of each 32-row slice the kernels read (offsets
    and values are kernel parameters)."""

    def __init__(self, n: int, nnz_l: int, nnz_u: int, val_bytes: int = 8, stencil: bool = False):
        self.n = n
        self.V = 8 * n
        self.stencil = stencil
        if stencil:
            self.ML = self.MU = 32 * ((n + 31) // 32)
        else:
            self.ML = (4 + val_bytes) * nnz_l + 4 * (n + 1)
            self.MU = (4 + val_bytes) * nnz_u + 4 * (n + 1)

    def spmv(self):
        return self.ML + self.MU + 3 * self.V

    def gs2_sweep(self, n_j: int):
        V, ML, MU = self.V, self.ML, self.MU
        b = ML + MU + 4 * V
        if n_j == 1:
            b += ML + 3 * V
        elif n_j >= 2:
            b += (ML + 2 * V) + (n_j - 2) * (ML + 3 * V) + (ML + 4 * V)
        return b

    def precond_gs2_zero_start(self, n_j: int):
        """GS2(1,1,n_j) from z = 0: the residual pass is elided (b - A*0 == b)."""
        V, ML = self.V, self.ML
        if n_j == 0:
            return 3 * V
        if n_j == 1:
            return ML + 3 * V
        return (ML + 3 * V) + (n_j - 2) * (ML + 3 * V) + (ML + 4 * V)

    def cgs2(self, k: int):
        return 2 * (2 * k + 3) * self.V

    def arnoldi_step(self, j: int, n_j: int):
        return self.precond_gs2_zero_start(n_j) + self.spmv() + self.cgs2(j + 1) + 2 * self.V

    def cycle(self, m: int, n_j: int):
        steps = sum(self.arnoldi_step(j, n_j) for j in range(m))
        end = (m + 1) * self.V + self.precond_gs2_zero_start(n_j) + 3 * self.V + self.spmv() + 3 * self.V
        return steps + end

    # bytes the executed fused kernels must move (for their rooflines), k = basis rows in the pass
    def dcgs_dots(self, k: int):
        return (k + 1) * self.V            # V rows [0, k) + w

    def dcgs_update(self, k: int):
        return (k + 1) * self.V + 2 * self.V  # V rows [0, k) + w read; v_j and u' written

    def cgs_dots(self, k: int):
        return (k + 1) * self.V

    def cgs_update(self, k: int):
        return (k + 2) * self.V            # V rows + w read, w written

    def step_actual(self, j: int, n_j: int, ortho: str = "dcgs2"):
        """Algorithmic bytes the B200 kernels move for Arnoldi iteration j (zero-start preconditioner,
        SpMV, fused orthogonalisation passes over the k = j + 1 basis rows, 2V of vector passes)."""
        k = j + 1
        orth = (self.dcgs_dots(k) + self.dcgs_update(k)) if ortho == "dcgs2" else \
            (self.cgs_dots(k) + 2 * self.cgs_update(k))
        return self.precond_gs2_zero_start(n_j) + self.spmv() + 2 * self.V + orth

    def cycle_end_actual(self, m: int, n_j: int, ortho: str = "dcgs2"):
        """Cycle end: the last column's dots (DCGS2), V^T-combination, preconditioner, update, SpMV,
        residual."""
        V = self.V
        last = self.dcgs_dots(m + 1) if ortho == "dcgs2" else 0
        return last + (m + 2) * V + self.precond_gs2_zero_start(n_j) + 3 * V + self.spmv() + 3 * V

    def cycle_actual(self, m: int, n_j: int, ortho: str = "dcgs2"):
        """Algorithmic bytes of the kernels one cycle actually launches (value's numerator)."""
        return sum(self.step_actual(j, n_j, ortho) for j in range(m)) + self.cycle_end_actual(m, n_j, ortho)

    def step_mgs_own(self, j: int, n_j: int):
        """Bytes of the reference's own MGS Arnoldi iteration j (oracle): per basis vector one dot
        (2V) and one update (3V), then norm (V) and scaling (2V)."""
        return self.precond_gs2_zero_start(n_j) + self.spmv() + (j + 1) * 5 * self.V + 3 * self.V


def laplace3d_nnz(nx, ny, nz):
    n = nx * ny * nz
    nnz_l = (nx - 1) * ny * nz + nx * (ny - 1) * nz + nx * ny * (nz - 1)
    return n, nnz_l, nnz_l


# ---------------------------------------------------------------- environment helpers
def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.rows.append([c.strip() for c in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        pw = [float(r[3]) for r in self.rows if r[3].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "power_w_max": max(pw) if pw else None}


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(
        os.environ.get("LOCAL_RANK", "0"))


# ---------------------------------------------------------------- CPU baseline (oracle port)
class CpuSample:
    """The C oracle (the reference algorithm: MGS GMRES(60) with the zero-start GS2(1,1,1)
    preconditioner) on laplace3d nx^3, sampled one Arnoldi iteration at a time.

    A GMRES(60) cycle's cost depends on the iteration index j (the MGS loop runs over j + 1 basis
    vectors), so a bounded sample of the workload is a set of iterations j drawn stratified across
    the cycle (j_s = floor((s + 1/2) m / K) for K samples): the sample has the cycle's j-mix.  The
    basis rows are pseudo-random unit vectors (the cost of an iteration does not depend on their
    values).  Setup (host CSR, splitting, basis) is excluded from timing, like the reference CLI
    (cli.py:162-176)."""

    def __init__(self, nx: int, threads: int, m: int = 60):
        import numpy as np

        import oracle
        from paper_2104_01196_b200 import problems

        self.np = np
        self.oracle = oracle
        oracle.set_threads(threads)
        oracle.set_dot_threads(threads)
        self.threads = threads
        self.nx = nx
        self.m = m
        a = problems.laplace3d(nx)
        self.mat = oracle.Matrix(a)
        self.mat.split()
        n = a.nrows
        self.b = oracle.random_rhs(n, 0)
        self.pre = oracle.Precond(self.mat, "gs2", n_t=1, n_k=1, n_j=1)
        self.V = np.empty((m + 1, n))
        for i in range(m + 1):
            v = oracle.random_rhs(n, 1000 + i)
            self.V[i] = v / np.sqrt(oracle.dot(v, v))
        self.w = np.empty(n)
        self.z = np.empty(n)
        n_, nl, nu = laplace3d_nnz(nx, nx, nx)
        # the B200 arm's byte count for the same work: laplace3d's triangles are stencil-encoded there
        self.mod = Model(n_, nl, nu, stencil=True)

    def js(self, k: int):
        return [min(self.m - 1, int((s + 0.5) * self.m / k)) for s in range(k)]

    def step(self, j: int) -> float:
        t0 = time.perf_counter()
        self.oracle.arnoldi_step(self.mat, self.pre, self.V, j, self.w, self.z)
        return time.perf_counter() - t0

    def work(self, j: int) -> int:
        """The B200 path's algorithmic bytes for iteration j (the common numerator of both arms)."""
        return self.mod.step_actual(j, 1)

    def sweeps(self, reps: int = 2):
        """Per-sweep ms of the reference's relaxations (a6-a8) on b = rhs(0), x = rhs(1): the
        SURVEY §8(d) CPU timing (median of reps, 1 application each)."""
        o, m = self.oracle, self.mat
        x1 = o.random_rhs(m.n, 1)
        out = {}

        def med(fn):
            ts = []
            for _ in range(reps):
                x = x1.copy()
                t0 = time.perf_counter()
                fn(x)
                ts.append((time.perf_counter() - t0) * 1e3)
            return round(statistics.median(ts), 1)

        out["gs2_nj1_ms"] = med(lambda x: o.gs2_apply(m, self.b, x, n_t=1, n_k=1, n_j=1))
        out["jr_ms"] = med(lambda x: o.jr_sweeps(m, self.b, x, 1))
        out["gs_seq_ms"] = med(lambda x: o.gs_sweep(m, self.b, x, "forward"))
        out["spmv_ms"] = med(lambda x: o.spmv(m, x))
        return out


def reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    n_gpus = max(world, args.gpus)
    threads = os.cpu_count() or 1
    # the sample is always laplace3d 256^3: the C5 workload (512^3, N > 1) needs > 64 GB of host RAM
    # for the CPU matrix + splitting + basis (measured: killed at 62 GB); W per row is the same at
    # both sizes (the slab per GPU at N = 8 is the 256^3 problem)
    nx = args.ref_nx
    target = f"laplace3d {nx}^3 (C2)" if n_gpus == 1 else "laplace3d 512^3 (C5), sampled on a 256^3 instance"
    cs = CpuSample(nx, threads)
    for j in cs.js(max(args.warmup, 1))[: args.warmup]:
        cs.step(j)
    js = cs.js(args.steps)
    ts = [cs.step(j) for j in js]
    work = sum(cs.work(j) for j in js)
    own = sum(cs.mod.step_mgs_own(j, 1) for j in js)
    secs = sum(ts)
    v = work / secs / 1e9
    m = cs.m
    # a full cycle = the 60 iterations (+ its end); the stratified sample's mean iteration time
    # estimates ms per cycle
    ms_cycle = secs / len(js) * m * 1e3
    sample = (f"C oracle (reference algorithm: MGS GMRES(60) + zero-start GS2(1,1,1)), Arnoldi iterations "
              f"j = {js[0]}..{js[-1]} stratified over the 60-step cycle of laplace3d {nx}^3 (one per step, "
              f"{secs:.1f} s total), {threads} host threads (OpenMP row loops, threaded ddot split), setup excluded")
    line = {
        "metric": METRIC, "value": round(v, 3), "unit": "GB/s", "n_gpus": n_gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_cycle, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{target}: GMRES(60) + GS2(1,1,1) preconditioner (bounded sample of the cycle)",
                   "sample": sample, "iterations_sampled": js,
                   "work_note": "value = the B200 path's algorithmic bytes for the sampled iterations / CPU time "
                                "(the same numerator as the GPU arm, so the ratio is a time ratio on identical "
                                "work); own_gbs = the oracle's own MGS bytes / time",
                   "own_gbs": round(own / secs / 1e9, 3),
                   "ms_per_iteration": round(secs / len(js) * 1e3, 2)},
        "impl": "reference",
        "cpu_baseline": {"value": round(v, 3), "unit": "GB/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- GPU arm
def ours(args):
    import torch

    import paper_2104_01196_b200 as g2
    from paper_2104_01196_b200 import _native
    from paper_2104_01196_b200.krylov import KernelTimer

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        from paper_2104_01196_b200 import distributed as gd

        return gd.bench_rank(args, METRIC, Model, laplace3d_nnz, ClockSampler, peaks)

    lib = _native.load()
    nx = args.nx or 256
    n_j = 1
    m = args.restart
    setup = {}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a = g2.laplace3d(nx, device=local)  # on-device stencil build + split-CSR (SELL-32) + D^-1 scaling
    torch.cuda.synchronize()
    setup["device_matrix_build_split_s"] = round(time.perf_counter() - t0, 4)
    n = a.nrows
    b = g2.random_rhs(n, 0, device=f"cuda:{local}")
    pc = g2.Preconditioner(a, "gs2", g2.RelaxConfig(1, 1, n_j))
    layout = {"L": a.layout(0), "U": a.layout(1)}
    stencil = layout["L"]["stencil_k"] > 0 and layout["U"]["stencil_k"] > 0
    mod = Model(n, a.nnz_l, a.nnz_u, stencil=stencil)
    mod_csr = Model(n, a.nnz_l, a.nnz_u)
    actual_bytes = mod.cycle_actual(m, n_j)
    model_bytes = mod_csr.cycle(m, n_j)
    hbm, peak_kind = peaks()

    def step():
        g2.gmres(a, b, pc, restart=m, tol=1e-300, maxit=m)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = lib.rs_launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
    launches = lib.rs_launch_count() - l0
    ms = e0.elapsed_time(e1) / args.steps
    value = actual_bytes / (ms * 1e-3) / 1e9

    # per-kernel-group attribution inside one more (instrumented) cycle
    with KernelTimer() as kt:
        step()
    ksum = kt.summary()
    group_bytes = {
        "precond": (m + 1) * mod.precond_gs2_zero_start(n_j),
        "spmv": (m + 2) * mod.spmv(),
        "cgs_dots": sum(mod.cgs_dots(k) for k in range(1, m + 1)),
        "cgs_update_dots": sum(mod.cgs_update(k) for k in range(1, m + 1)),
        "cgs_update_norm": sum(mod.cgs_update(k) for k in range(1, m + 1)),
        # DCGS2 (default ortho): dual dots over rows [0, k) for k = 1..m+1 (the last one only
        # finalises the last column), update over rows [0, k) for k = 1..m
        "dcgs_dots": sum(mod.dcgs_dots(k) for k in range(1, m + 2)),
        "dcgs_update": sum(mod.dcgs_update(k) for k in range(1, m + 1)),
        "scale": m * 2 * mod.V,
    }
    total_ms = sum(t for _, t in ksum.values())
    kernels = {}
    for g, (cnt, t) in ksum.items():
        gb = group_bytes.get(g)
        kernels[g] = {"launches": cnt, "ms": round(t, 3), "share": round(t / total_ms, 3) if total_ms else None,
                      "gbs": round(gb / (t * 1e-3) / 1e9, 1) if gb and t else None,
                      "bytes_per_launch": round(gb / cnt) if gb and cnt else None}
    dom = max((g for g in kernels if g in group_bytes), key=lambda g: kernels[g]["ms"])
    # traffic: ncu DRAM bytes of one launch of the dominant kernel (profiles/traffic.json, stamped with
    # the git sha of the capture), scaled to this cycle's average launch by the measured traffic /
    # algorithmic-bytes ratio of that launch
    traffic, traffic_src = None, None
    tfile = ROOT / "profiles" / "traffic.json"
    if tfile.exists():
        tj = json.loads(tfile.read_text())
        t = tj.get(dom)
        if t:
            ratio = (t["dram_read"] + t["dram_write"]) / t["model_bytes"]
            traffic = round(ratio * group_bytes[dom] / kernels[dom]["launches"])
            traffic_src = f"profiles/traffic.json ({t.get('capture', '?')}, sha {tj.get('git_sha', '?')})"
    roofline = {"bound": "hbm", "kernel": dom, "achieved": kernels[dom]["gbs"], "peak": hbm, "unit": "GB/s",
                "frac": round(kernels[dom]["gbs"] / hbm, 3), "traffic": traffic, "traffic_source": traffic_src,
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                "achieved_note": "algorithmic bytes of the group's launches (SURVEY §8(d) per-row figures x rows) / "
                                 "the group's CUDA-event time on the launching stream",
                "cycle_frac": round(value / hbm, 3)}

    # e2e through the public API with host buffers: pinned b in, x out
    b_host = b.cpu().pin_memory()
    x = None
    for _ in range(args.warmup):  # untimed: first-touch of the pinned output blocks (the caller keeps the
        x = g2.gmres(a, b_host, pc, restart=m, tol=1e-300, maxit=m)[0]  # previous x alive, as in the timed loop)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_steps = []
    for _ in range(args.steps):
        ts = time.perf_counter()
        x = g2.gmres(a, b_host, pc, restart=m, tol=1e-300, maxit=m)[0]
        assert not x.is_cuda
        e2e_steps.append(round((time.perf_counter() - ts) * 1e3, 2))
    e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    e2e = {"value": round(actual_bytes / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": 8 * n,
           "d2h_bytes_per_step": 8 * n, "ms_per_step": round(e2e_ms, 3), "ms_steps": e2e_steps}

    sweeps = sweep_table(g2, torch, a, mod, hbm, setup, mod_csr=mod_csr) if not args.no_sweeps else None
    tts = None
    if not args.no_tts:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, h = g2.gmres(a, b, pc, restart=m, tol=1e-9)
        torch.cuda.synchronize()
        tts = {"seconds": round(time.perf_counter() - t0, 3), "iterations": h.iterations, "converged": h.converged,
               "final_rel_res": h.final_rel_res, "preconditioner": "gs2(1,1,1)", "restart": m, "tol": 1e-9,
               "reference_iterations": 2635, "reference_seconds_1core": 11002,
               "note": "default ortho (DCGS2, fixed-order device reductions); ortho='mgs_ref' reproduces the "
                       "reference's history bitwise (profiles/r02_c2_mgs_ref.json)"}
    # C5 on ONE GPU: the 512^3 cycle, the strong-scaling reference for the N > 1 lines (which run
    # 512^3 in z-slabs); the 256^3 workspace is released first (512^3 basis: 65.5 GB)
    c5 = None
    if not args.no_c5 and (args.nx or 256) == 256:
        from paper_2104_01196_b200 import krylov as gk

        del a, pc
        gk.release_workspace()
        torch.cuda.empty_cache()
        a5 = g2.laplace3d(512, device=local)
        b5 = g2.random_rhs(a5.nrows, 0, device=f"cuda:{local}")
        pc5 = g2.Preconditioner(a5, "gs2", g2.RelaxConfig(1, 1, n_j))
        mod5 = Model(a5.nrows, a5.nnz_l, a5.nnz_u, stencil=a5.layout(0)["stencil_k"] > 0)
        g2.gmres(a5, b5, pc5, restart=m, tol=1e-300, maxit=m)
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(2):
            g2.gmres(a5, b5, pc5, restart=m, tol=1e-300, maxit=m)
        f1.record()
        torch.cuda.synchronize()
        ms5 = f0.elapsed_time(f1) / 2
        c5 = {"workload": "C5 laplace3d 512^3 on ONE GPU, one GMRES(60) cycle (strong-scaling reference of the "
                          "N > 1 lines)", "ms_per_step": round(ms5, 3),
              "value": round(mod5.cycle_actual(m, n_j) / (ms5 * 1e-3) / 1e9, 3), "unit": "GB/s"}
        del a5, b5, pc5
        gk.release_workspace()
        torch.cuda.empty_cache()
    configs = None
    if not args.no_configs:
        configs = secondary_configs(g2, torch)
    cpu = None
    if not args.no_cpu_baseline:
        cs = CpuSample(nx, 1)
        js = cs.js(3)
        secs = sum(cs.step(j) for j in js)
        cpu = {"value": round(sum(cs.work(j) for j in js) / secs / 1e9, 3), "unit": "GB/s", "cores": 1,
               "kind": "port",
               "sample": f"C oracle (reference algorithm), Arnoldi iterations j = {js} of the GMRES(60)+GS2(1,1,1) "
                         f"cycle on laplace3d {nx}^3, 1 host core, {secs:.1f} s (value: the B200 path's bytes for "
                         f"that work / CPU time, as in the reference arm)",
               "own_gbs": round(sum(cs.mod.step_mgs_own(j, 1) for j in js) / secs / 1e9, 3),
               "per_sweep_ms_1core": cs.sweeps()}
        del cs
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C2: laplace3d {nx}^3 ({n} rows), one GMRES({m}) cycle with GS2(1,1,1) "
                               f"zero-start preconditioner, b = random_rhs(n, 0)",
                   "ortho": "dcgs2 (CGS2 with delayed re-orthogonalisation, 2 basis passes per step)",
                   "bytes_per_step": actual_bytes,
                   "matrix_layout": layout,
                   "bytes_note": "value = algorithmic bytes of the launched kernel sequence (fused passes counted "
                                 "once) / device time: the whole-cycle HBM throughput",
                   "model_bytes_per_step": model_bytes,
                   "model_gbs": round(model_bytes / (ms * 1e-3) / 1e9, 1),
                   "model_note": "SURVEY §8(d) model of the cycle (split-CSR matrix bytes, unfused CGS2, 4 basis "
                                 "reads per step): a fixed work figure; with the stencil-encoded triangles and the "
                                 "fused DCGS2 passes the kernels move fewer bytes, so model_gbs exceeds the HBM peak; "
                                 "work figure, exceeds the HBM peak because the fused kernels move fewer bytes",
                   "ms_per_iteration": round(ms / m, 4),
                   "iterations_per_s": round(m / (ms * 1e-3), 1),
                   "row_iterations_per_s": round(n * m / (ms * 1e-3)),
                   "l2": "inputs larger than L2 (V basis 61 x 134 MB, vectors 134 MB each)", "parallelism": "1 GPU",
                   "scaling_note": "N > 1 lines run C5 (laplace3d 512^3 in N z-slabs, fixed total problem); the "
                                   "512^3 cycle on this one GPU is c5_one_gpu"},
        "roofline": roofline, "kernels": kernels, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
        "clocks": clk.summary(), "sweeps": sweeps, "tts": tts, "c5_one_gpu": c5, "configs": configs,
        "setup": setup,
    }
    print(json.dumps(line), flush=True)
    return 0


def _timed(torch, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t0


def secondary_configs(g2, torch):
    """The other BASELINE.json configs, one compact record each (bench_configs.py has the full
    tables): C1 (laplace2d 128^2, GMRES(30): GS2(2,1,1) vs sequential GS(2); the reference's
    counts 563 / 471), C3 (elasticity3d 64^3: 50 stand-alone applications of JR(w=1) -- diverges --
    and GS2 n_j = 1/3/10 through stationary_solve, plus GMRES(60) counts), C4 (convdiff3d 256^3:
    fp64 vs fp32-inside-fp64 GS2(1,1,2) in GMRES(60))."""
    out = {}
    a = g2.laplace2d(128)
    b = g2.random_rhs(a.nrows, 0)
    c1 = {"workload": "C1 laplace2d 128^2, GMRES(30)", "reference_iterations": {"gs2(2,1,1)": 563, "gs_seq(2)": 471}}
    for label, kind, cfg in (("gs2(2,1,1)", "gs2", (2, 1, 1)), ("gs_seq(2)", "gs_seq", (2, 1, 0))):
        pm = g2.Preconditioner(a, kind, g2.RelaxConfig(*cfg))
        g2.gmres(a, b, pm, restart=30)
        (_, h), dt = _timed(torch, lambda: g2.gmres(a, b, pm, restart=30))
        c1[label] = {"iterations": h.iterations, "seconds": round(dt, 4)}
    if hasattr(g2, "stationary_solve"):
        pm_cfg = g2.RelaxConfig(2, 1, 1)
        g2.stationary_solve(a, b, "gs2", pm_cfg, tol=1e-6, maxit=50)
        (_, h), dt = _timed(torch, lambda: g2.stationary_solve(a, b, "gs2", pm_cfg, tol=1e-6))
        c1["stationary gs2(2,1,1) to 1e-6"] = {"applications": h.iterations, "final_rel_res": h.final_rel_res,
                                               "seconds": round(dt, 4), "reference_applications": 8872,
                                               "reference_seconds_1core": 9.9}
    out["c1"] = c1
    t0 = time.perf_counter()
    a = g2.elasticity3d(64)
    gen = time.perf_counter() - t0
    b = g2.random_rhs(a.nrows, 0, device="cuda")
    c3 = {"workload": f"C3 elasticity3d 64^3 (n = {a.nrows}, nnz = {a.nnz})", "host_generation_s": round(gen, 1)}
    if hasattr(g2, "stationary_solve"):
        st = {}
        for label, kind, cfg in (("jr(w=1)", "jr", (1, 1, 0)), ("gs2 n_j=1", "gs2", (1, 1, 1)),
                                 ("gs2 n_j=3", "gs2", (1, 1, 3)), ("gs2 n_j=10", "gs2", (1, 1, 10))):
            g2.stationary_solve(a, b, kind, g2.RelaxConfig(*cfg), tol=1e-300, maxit=2)  # warm-up (buffers)
            (_, h), dt = _timed(torch, lambda: g2.stationary_solve(a, b, kind, g2.RelaxConfig(*cfg), tol=1e-300,
                                                                   maxit=50))
            st[label] = {"applications": h.iterations, "rel_res": h.final_rel_res,
                         "ms_per_application": round(dt * 1e3 / max(h.iterations, 1), 3)}
        c3["stationary_50"] = st
        c3["reference_rel_res_50"] = {"jr(w=1)": 3.40e9, "gs2 n_j=1": 71.1, "gs2 n_j=3": 5.92e-2, "gs2 n_j=10": 4.46e-3}
    gm = {}
    for label, kind, cfg in (("gs2 n_j=1", "gs2", (1, 1, 1)), ("gs2 n_j=3", "gs2", (1, 1, 3))):
        pm = g2.Preconditioner(a, kind, g2.RelaxConfig(*cfg))
        (_, h), dt = _timed(torch, lambda: g2.gmres(a, b, pm, restart=60, maxit=3000))
        gm[label] = {"iterations": h.iterations, "converged": h.converged, "seconds": round(dt, 3)}
    c3["gmres60"] = gm
    out["c3"] = c3
    del a, b
    a = g2.convdiff3d(256, (50.0, 25.0, 10.0), device="cuda")
    b = g2.random_rhs(a.nrows, 0, device="cuda")
    c4 = {"workload": "C4 convdiff3d 256^3 beta=(50,25,10), GMRES(60) + GS2(1,1,2)"}
    for prec in ("same", "single_inside_double"):
        pm = g2.Preconditioner(a, "gs2", g2.RelaxConfig(1, 1, 2), precision=prec)
        g2.gmres(a, b, pm, restart=60, maxit=60)
        (_, h), dt = _timed(torch, lambda: g2.gmres(a, b, pm, restart=60))
        c4[prec] = {"iterations": h.iterations, "converged": h.converged, "seconds": round(dt, 3),
                    "ms_per_iteration": round(dt * 1e3 / max(h.iterations, 1), 4)}
    out["c4"] = c4
    from paper_2104_01196_b200 import krylov as gk

    del a, b, pm
    gk.release_workspace()
    torch.cuda.empty_cache()
    return out


def sweep_table(g2, torch, a, mod, hbm, setup=None, reps: int = 10, mod_csr=None):
    """Same-device comparison of the paper's relaxations on x != 0 (b = rhs(0), x = rhs(1)).
    ``setup`` receives the one-off analysis costs the baselines pay (level sets, colouring).
    The GS2 / JR / SpMV rows run on the handle's default layout (stencil-encoded triangles for
    laplace3d, bytes from ``mod``) and again on the explicit SELL slots (``explicit``: the
    split-CSR kernels every non-stencil matrix runs, bytes from ``mod_csr``)."""
    n = a.nrows
    dev = a.torch_device
    b = g2.random_rhs(n, 0, device=dev)
    x0 = g2.random_rhs(n, 1, device=dev)
    s = g2.extract_splitting(a)
    out = {}

    def timeit(fn, nbytes, setup_key=None):
        x = x0.clone()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn(x)  # warm-up (builds level sets etc.)
        torch.cuda.synchronize()
        if setup_key and setup is not None:
            setup[setup_key] = round(time.perf_counter() - t0, 4)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn(x)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        r = {"ms": round(ms, 4)}
        if nbytes:
            r["gb"] = round(nbytes / 1e9, 4)
            r["gbs"] = round(nbytes / (ms * 1e-3) / 1e9, 1)
            r["frac"] = round(nbytes / (ms * 1e-3) / 1e9 / hbm, 3)
        return r

    y = torch.empty_like(b)

    def streaming_rows(md):
        rows = {}
        for nj in range(4):
            cfg = g2.RelaxConfig(1, 1, nj)
            rows[f"gs2_nj{nj}"] = timeit(lambda x, cfg=cfg: g2.gs2_apply(a, s, b, x, cfg), md.gs2_sweep(nj))
        rows["jr"] = timeit(lambda x: g2.jr_sweeps(a, s, b, x, 1), md.gs2_sweep(0))
        rows["spmv"] = timeit(lambda x: g2.spmv(a, x, out=y), md.spmv())
        return rows

    out.update(streaming_rows(mod))
    if mod_csr is not None and mod.stencil:
        a.set_diagonal_slices(False)
        try:
            out["explicit"] = streaming_rows(mod_csr)
            out["explicit"]["note"] = "same sweeps on the explicit SELL-32 slots (split-CSR bytes)"
        finally:
            a.set_diagonal_slices(True)
    out["layout_note"] = ("default rows: " + ("stencil-encoded triangles (lane masks per slice; bytes = vectors + "
                                              "masks)" if mod.stencil else "explicit SELL-32 slots"))
    out["gs_level_sched"] = timeit(lambda x: g2.gs_sequential_sweep(a, s, b, x, "forward"),
                                   (mod_csr or mod).ML + (mod_csr or mod).MU + 3 * mod.V,
                                   "level_set_analysis_plus_first_sweep_s")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    coloring = g2.greedy_color(a)
    torch.cuda.synchronize()
    if setup is not None:
        setup["greedy_coloring_s"] = round(time.perf_counter() - t0, 4)
    out["mt_gs"] = timeit(lambda x: g2.mt_gs_sweep(a, s, coloring, b, x, "forward"),
                          (mod_csr or mod).ML + (mod_csr or mod).MU + 3 * mod.V,
                          "mt_colour_ordered_slices_plus_first_sweep_s")
    out["mt_gs"]["colors"] = coloring.num_colors
    # smoother mode (row a14): GS2(1,1,1) applications WITH the per-application residual history
    # (fused into the next application's residual pass); compare with gs2_nj1 (no history)
    cfg1 = g2.RelaxConfig(1, 1, 1)
    g2.stationary_solve(a, b, "gs2", cfg1, tol=1e-300, maxit=4, x0=x0)
    torch.cuda.synchronize()
    napp = 256
    t0 = time.perf_counter()
    _, hs = g2.stationary_solve(a, b, "gs2", cfg1, tol=1e-300, maxit=napp, x0=x0)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / napp
    out["stationary_gs2_nj1"] = {"ms_per_application": round(ms, 4), "applications": hs.iterations,
                                 "gbs": round(mod.gs2_sweep(1) / (ms * 1e-3) / 1e9, 1),
                                 "frac": round(mod.gs2_sweep(1) / (ms * 1e-3) / 1e9 / hbm, 3),
                                 "note": "host wall time per application of a 256-application stationary_solve "
                                         "(batched, residual norm of every iterate recorded; includes the "
                                         "reference-order ||b||, a ~4 ms latency-bound recurrence, once per "
                                         "solve), GS2 sweep bytes"}
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--nx", type=int, default=0)
    p.add_argument("--restart", type=int, default=60)
    p.add_argument("--no-tts", action="store_true")
    p.add_argument("--tts", action="store_true", help="(default now) time a full solve at N > 1 as well")
    p.add_argument("--no-sweeps", action="store_true")
    p.add_argument("--comm", default="peer", choices=["peer", "nccl"],
                   help="N > 1 collectives: NVLink peer-memory kernels (default) or NCCL")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-c5", action="store_true", help="skip the 512^3 one-GPU cycle (strong-scaling reference)")
    p.add_argument("--ref-nx", type=int, default=256, help="(testing) grid of the reference arm's sample")
    p.add_argument("--no-configs", action="store_true", help="skip the C1 / C3 / C4 records of the N = 1 line")
    args = p.parse_args()
    if args.impl == "reference":
        return reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args.gpus)
    return ours(args)


def relaunch(n: int) -> int:
    """``--gpus N`` without a launcher: re-execute this script under torch.distributed.run with N
    ranks on this node (rendezvous on 127.0.0.1); rank 0 prints the JSON line."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "4")
    return subprocess.call(cmd, env=env)


if __name__ == "__main__":
    sys.exit(main())
