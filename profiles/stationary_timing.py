import sys, time, torch
sys.path.insert(0, "/root/repo")
import paper_2104_01196_b200 as g2
a = g2.laplace3d(256, device=0)
b = g2.random_rhs(a.nrows, 0, device="cuda:0"); x0 = g2.random_rhs(a.nrows, 1, device="cuda:0")
cfg = g2.RelaxConfig(1, 1, 1)
g2.stationary_solve(a, b, "gs2", cfg, tol=1e-300, maxit=4, x0=x0); torch.cuda.synchronize()
for _ in range(2):
    t0 = time.perf_counter(); _, h = g2.stationary_solve(a, b, "gs2", cfg, tol=1e-300, maxit=64, x0=x0); torch.cuda.synchronize()
    print("ms/app", (time.perf_counter() - t0) * 1e3 / 64, h.iterations)
import ctypes as C
from paper_2104_01196_b200 import _native as N
lib = N.load(); st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
scal = torch.zeros(2, dtype=torch.float64, device="cuda:0")
def tm(fn, reps=3):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) * 1e3 / reps
print("dot_blas ms", tm(lambda: lib.rs_dot_blas(a.nrows, C.c_void_p(b.data_ptr()), C.c_void_p(b.data_ptr()), C.c_void_p(scal.data_ptr()), 0, st)))
norms = torch.empty(65, dtype=torch.float64, device="cuda:0")
c = N.RelaxCfg.of(cfg); x = x0.clone()
for k in (1, 8, 64):
    ms = tm(lambda: lib.rs_stationary_batch(a.handle, N.PC_KINDS["gs2"], C.byref(c), C.c_void_p(b.data_ptr()), C.c_void_p(x.data_ptr()), k, C.c_void_p(norms.data_ptr()), st))
    print("batch", k, "ms", ms, "per app", ms / k)
print("gs2 sweep ms", tm(lambda: g2.gs2_apply(a, g2.extract_splitting(a), b, x, cfg), 10))
