"""dev: MINRES per-iteration device time (fixed 30 iterations after a warm-up) on box meshes with
both S^-1 — config 4 (128^3 p=4) and config 5 (graded two-material boxes)."""
import sys
sys.path.insert(0, ".")
import torch
from synth import make_config
from paper_2304_12387_b200 import from_problem
for name, p in [("c4", 4), ("c5", 4)]:
    pr = make_config(name, p=p)
    for schur in ("chebyshev", "amg"):
        op = from_problem(pr, schur=schur, amg_cheb_degree=1)
        b = torch.rand(op.sizes.n, dtype=torch.float64, device="cuda")
        op.minres(b, rtol=1e-30, maxit=6)
        _, rep = op.minres(b, rtol=1e-30, maxit=30)
        print(f"{name} {schur}: {rep.t_solve_ms / rep.iters:.3f} ms/it", flush=True)
        op.close()
        del b
        torch.cuda.empty_cache()
