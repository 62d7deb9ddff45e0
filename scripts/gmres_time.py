"""GMRES + block-triangular vs MINRES + block-diagonal time-to-solve (development aid)."""
import sys
sys.path.insert(0, ".")
import torch
from synth import make_config
from paper_2304_12387_b200 import from_problem

for name, N, p, m in [("c2", None, None, 30), ("c5", None, 4, 30), ("c3", None, None, 20)]:
    pr = make_config(name, N=N, p=p)
    op = from_problem(pr, schur="amg")
    n = op.sizes.n
    g = torch.Generator(device="cuda").manual_seed(1)
    xs = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    b = op.apply_block(xs)
    x, r1 = op.minres(b, rtol=1e-12, maxit=5000)
    e1 = ((x - xs).abs().max() / xs.abs().max()).item()
    x2, r2 = op.gmres(b, rtol=1e-12, maxit=5000, restart=m)
    e2 = ((x2 - xs).abs().max() / xs.abs().max()).item()
    print(f"{name} p={pr.p} n={n}: MINRES+diag {r1.iters} its {r1.t_solve_ms:.1f} ms err {e1:.1e} | "
          f"GMRES({m})+tri {r2.iters} its {r2.t_solve_ms:.1f} ms err {e2:.1e}", flush=True)
    op.close(); del x, x2, b, xs; torch.cuda.empty_cache()
