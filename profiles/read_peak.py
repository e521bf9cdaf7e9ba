"""Pure-read and copy bandwidth on this B200 (torch reductions / copies, CUDA events): the ceiling the
read-dominated DCGS2 passes work against (MEASURED_PEAKS.json holds the copy figure)."""
import torch
x = torch.empty(1 << 30, dtype=torch.float64, device="cuda")  # 8 GiB
x.uniform_()
y = torch.empty_like(x)
def tm(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
ms = tm(lambda: x.sum()); print("read (sum) GB/s", round(8 * 2**30 / ms / 1e6, 1))
ms = tm(lambda: torch.dot(x, x)); print("read (dot) GB/s", round(8 * 2**30 / ms / 1e6, 1))
ms = tm(lambda: y.copy_(x)); print("copy GB/s (r+w)", round(2 * 8 * 2**30 / ms / 1e6, 1))
