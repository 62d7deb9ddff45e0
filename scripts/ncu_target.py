"""Small driver for ncu captures: build one operator and run a few applies.
    python scripts/ncu_target.py [config] [p] [n_applies] [kernel]"""
import sys
sys.path.insert(0, ".")
import torch
from synth import make_config
from paper_2304_12387_b200 import from_problem

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
p = int(sys.argv[2]) if len(sys.argv) > 2 else 4
n = int(sys.argv[3]) if len(sys.argv) > 3 else 5
kern = int(sys.argv[4]) if len(sys.argv) > 4 else 0
pr = make_config(cfg, p=p)
op = from_problem(pr, kernel=kern, schur="chebyshev")
x = torch.rand(op.sizes.n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(n):
    op.apply_block(x, y)
torch.cuda.synchronize()
print("done", cfg, p, op.sizes.n)
