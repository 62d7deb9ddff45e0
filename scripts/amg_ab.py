"""dev: AMG MINRES timings for A/B (config 3 with the A9d polynomial, config 4 plain V-cycle)."""
import sys
sys.path.insert(0, ".")
import torch
from synth import make_config, random_vector
from paper_2304_12387_b200 import from_problem
for name, k in [("c3", 3), ("c4", 1)]:
    pr = make_config(name)
    op = from_problem(pr, schur="amg", amg_cheb_degree=k)
    b = torch.from_numpy(random_vector(op.sizes.n, 1)).cuda()
    op.minres(b, rtol=1e-12, maxit=6)
    x, rep = op.minres(b, rtol=1e-12, maxit=4000)
    print(f"{name} k={k}: {rep.iters} its {rep.t_solve_ms:.1f} ms ({rep.t_solve_ms / rep.iters:.2f} ms/it)", flush=True)
    op.close()
    del b, x
    torch.cuda.empty_cache()
