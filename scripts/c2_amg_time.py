"""dev: config-2 MINRES time with both S^-1 (regression check)."""
import sys
sys.path.insert(0, ".")
import torch
from synth import make_config, random_vector
from paper_2304_12387_b200 import from_problem
pr2 = make_config("c2")
for schur in ("chebyshev", "amg"):
    op2 = from_problem(pr2, schur=schur)
    xs = torch.from_numpy(random_vector(op2.sizes.n, 2)).cuda()
    b = op2.apply_block(xs)
    for r in range(4):
        _, rep = op2.minres(b, rtol=1e-12, maxit=5000)
        print(schur, r, rep.iters, f"{rep.t_solve_ms:.2f} ms", flush=True)
    op2.close()
