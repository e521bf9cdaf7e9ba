"""Level-scheduled GS sweep timing + launch count (cooperative single launch vs per-level launches)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2104_01196_b200 as g2  # noqa: E402
from paper_2104_01196_b200 import _native  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 256
lib = _native.load()
a = g2.laplace3d(nx, device="cuda")
s = g2.extract_splitting(a)
b = g2.random_rhs(a.nrows, 0, device="cuda")
x = g2.random_rhs(a.nrows, 1, device="cuda")
g2.gs_sequential_sweep(a, s, b, x, "forward")
torch.cuda.synchronize()
l0 = lib.rs_launch_count()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    g2.gs_sequential_sweep(a, s, b, x, "forward")
e1.record()
torch.cuda.synchronize()
print({"nx": nx, "ms_per_sweep": e0.elapsed_time(e1) / 5, "launches_per_sweep": (lib.rs_launch_count() - l0) / 5,
       "err": _native.load().rs_last_error().decode()})
