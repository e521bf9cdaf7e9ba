import sys, torch
sys.path.insert(0, '/root/repo')
import paper_2104_01196_b200 as g2
a = g2.laplace3d(256, device=0); n = a.nrows
b = g2.random_rhs(n, 0, device="cuda:0"); x0 = g2.random_rhs(n, 1, device="cuda:0")
s = g2.extract_splitting(a); col = g2.greedy_color(a)
x = x0.clone(); g2.mt_gs_sweep(a, s, col, b, x, "forward"); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): g2.mt_gs_sweep(a, s, col, b, x, "forward")
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print({"mt_gs_ms": round(ms, 4), "gbs_model": round(1.7401e9 / ms / 1e6, 1), "colors": col.num_colors})
