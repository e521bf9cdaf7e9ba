"""ncu target: SpMV + GS2(1,1,1) preconditioner on laplace3d 256^3 with the matrix layout given on the
command line (stencil | dia | explicit; RS_SELL_STENCIL=0 selects dia for 'dia')."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2104_01196_b200 as g2  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "stencil"
a = g2.laplace3d(256, device=0)
if mode == "explicit":
    a.set_diagonal_slices(False)
x = g2.random_rhs(a.nrows, 1, device=a.torch_device)
y = torch.empty_like(x)
pc = g2.Preconditioner(a, "gs2", g2.RelaxConfig(1, 1, 1))
z = torch.empty_like(x)
for _ in range(3):
    g2.spmv(a, x, out=y)
    pc.apply_into(x, z)
torch.cuda.synchronize()
b = g2.random_rhs(a.nrows, 0, device=a.torch_device)
s = g2.extract_splitting(a)
g2.gs2_apply(a, s, b, y, g2.RelaxConfig(1, 1, 0))
g2.gs2_apply(a, s, b, y, g2.RelaxConfig(1, 1, 1))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
g2.spmv(a, x, out=y)
pc.apply_into(x, z)
g2.gs2_apply(a, s, b, y, g2.RelaxConfig(1, 1, 0))
g2.gs2_apply(a, s, b, y, g2.RelaxConfig(1, 1, 1))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
