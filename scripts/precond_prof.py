"""A few preconditioner applies at config 4 (ncu target for the S^-1 kernels)."""
import sys
sys.path.insert(0, ".")
import torch
from synth import make_config
from paper_2304_12387_b200 import from_problem
pr = make_config(sys.argv[1] if len(sys.argv) > 1 else "c4", p=4)
op = from_problem(pr, schur="chebyshev")
b = torch.rand(op.sizes.n, dtype=torch.float64, device="cuda")
z = torch.empty_like(b)
for _ in range(3):
    op.apply_precond(b, z)
torch.cuda.synchronize()
print("done")
