"""Reading A9d study: MINRES to 1e-12 with S^-1 = Chebyshev polynomial (degree k) in the AMG
V-cycle, on config 3 (64^3 p=4, contrast 1e4), its SPE10-shaped pure-Neumann variant and
config 4; iterations and device time-to-solve per degree."""
import sys
sys.path.insert(0, ".")
import torch
from synth import make_config, random_vector
from paper_2304_12387_b200 import from_problem

cases = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c3", "c3s", "c4"]
degs = [int(k) for k in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 3, 4]
ratio = float(sys.argv[3]) if len(sys.argv) > 3 else 20.0
sweeps = [int(k) for k in sys.argv[4].split(",")] if len(sys.argv) > 4 else [2]
for name in cases:
    pr = make_config(name)
    for k, nu in [(k, nu) for k in degs for nu in sweeps]:
        op = from_problem(pr, schur="amg", amg_cheb_degree=k, amg_cheb_ratio=ratio, amg_sweeps=nu)
        b = torch.from_numpy(random_vector(op.sizes.n, 1)).cuda()
        if pr.project_mean:
            b[op.sizes.n_rt:] -= b[op.sizes.n_rt:].mean()
        op.minres(b, rtol=1e-12, maxit=5)
        x, rep = op.minres(b, rtol=1e-12, maxit=4000)
        print(f"{name} k={k} nu={nu} ratio={ratio}: conv={rep.converged} {rep.iters} its "
              f"{rep.t_solve_ms:.1f} ms ({rep.t_solve_ms / max(rep.iters, 1):.2f} ms/it) "
              f"rel {rep.rel_resid:.2e}", flush=True)
        op.close()
        del b, x
        torch.cuda.empty_cache()
