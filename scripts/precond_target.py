"""ncu driver: a few preconditioner applies at config-4 size (development aid)."""
import sys
sys.path.insert(0, ".")
import torch
from synth import make_config
from paper_2304_12387_b200 import from_problem
p = int(sys.argv[1]) if len(sys.argv) > 1 else 4
op = from_problem(make_config("c4", p=p))
b = torch.rand(op.sizes.n, dtype=torch.float64, device="cuda")
z = torch.empty_like(b)
for _ in range(2):
    op.apply_precond(b, z)
torch.cuda.synchronize()
print("done")
