"""MINRES time-to-solve on the latency-bound configs (config 2, config 5 paper-scale), both S^-1
(development aid): python scripts/small_time.py"""
import sys
sys.path.insert(0, ".")
import torch
from synth import make_config, random_vector
from paper_2304_12387_b200 import from_problem

for name, p in [("c2", 3), ("c5", 2), ("c5", 4), ("c1", 2)]:
    pr = make_config(name, p=p)
    for schur in ("chebyshev", "amg"):
        op = from_problem(pr, schur=schur)
        b = op.apply_block(torch.from_numpy(random_vector(op.sizes.n, 2)).cuda())
        op.minres(b, rtol=1e-12, maxit=5000)
        best = None
        for _ in range(3):
            _, rep = op.minres(b, rtol=1e-12, maxit=5000)
            best = rep if best is None or rep.t_solve_ms < best.t_solve_ms else best
        print(f"{name} p={p} n={op.sizes.n} {schur:9s}: {best.iters} its {best.t_solve_ms:.2f} ms "
              f"({1e3 * best.t_solve_ms / max(best.iters, 1):.1f} us/it)", flush=True)
        op.close()
