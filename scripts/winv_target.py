"""ncu driver: the W^-1 (apply_z) path on the Table dg-mass-inv workload shape at order p."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from synth import make_config, random_vector
from paper_2304_12387_b200 import from_problem
p = int(sys.argv[1]) if len(sys.argv) > 1 else 4
ne = max(2, int(round((1.7e6 / p ** 3) ** (1.0 / 3.0))))
pr = make_config("c3", N=(ne, ne, ne), p=p)
pr.kind, pr.alpha, pr.beta = "grad_div", np.ones(pr.E), np.ones(pr.E)
op = from_problem(pr)
q = torch.from_numpy(random_vector(op.sizes.n_l2, 5)).cuda()
y = torch.empty_like(q)
for _ in range(4):
    op.apply_z(q, y)
torch.cuda.synchronize()
print("done", p, op.sizes.n_l2)
