"""MINRES per-iteration device time at BASELINE sizes (fixed iteration count, not converged)."""
import sys
sys.path.insert(0, ".")
import torch
from synth import make_config
from paper_2304_12387_b200 import from_problem

for name, p, N in [("c4", 4, None), ("c3", 4, None), ("c2", 3, None)]:
    pr = make_config(name, p=p, N=N)
    op = from_problem(pr, schur="chebyshev")
    b = torch.rand(op.sizes.n, dtype=torch.float64, device="cuda")
    op.minres(b, rtol=1e-12, maxit=12)
    x, rep = op.minres(b, rtol=1e-12, maxit=60)
    print(f"{name} p={p}: {rep.iters} its in {rep.t_solve_ms:.1f} ms -> {rep.t_solve_ms/max(rep.iters,1):.3f} ms/it "
          f"(rel {rep.rel_resid:.2e}), n={op.sizes.n}", flush=True)
    ys = torch.empty(op.sizes.n_l2, dtype=torch.float64, device="cuda")
    xs = torch.rand(op.sizes.n_l2, dtype=torch.float64, device="cuda")
    z = torch.empty_like(b)
    for _ in range(3): op.apply_precond(b, z)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10): op.apply_precond(b, z)
    e1.record(); torch.cuda.synchronize()
    print(f"   precond apply {e0.elapsed_time(e1)/10:.3f} ms", flush=True)
    op.close(); del b, x, z; torch.cuda.empty_cache()
