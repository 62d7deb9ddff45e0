"""MINRES time-to-solve with Chebyshev vs AMG S^-1 at BASELINE sizes (development aid)."""
import sys, time
sys.path.insert(0, ".")
import torch
from synth import make_config, random_vector
from paper_2304_12387_b200 import from_problem

cases = [("c2", None, None), ("c3", None, None), ("c5", None, 4), ("c4", None, 4)]
for name, N, p in cases:
    pr = make_config(name, N=N, p=p)
    for schur in ("chebyshev", "amg"):
        t0 = time.time()
        op = from_problem(pr, schur=schur)
        torch.cuda.synchronize()
        ts = time.time() - t0
        n = op.sizes.n
        g = torch.Generator(device="cuda").manual_seed(1)
        xs = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
        b = torch.empty_like(xs)
        op.apply_block(xs, b)
        maxit = 3000 if name != "c4" else 600
        x, rep = op.minres(b, rtol=1e-12, maxit=maxit)
        err = ((x - xs).abs().max() / xs.abs().max()).item()
        lv = op.amg_levels() if schur == "amg" else 0
        print(f"{name} p={pr.p} n={n} {schur:9s} levels={lv} setup {ts:.2f}s: {rep.iters} its "
              f"conv={rep.converged} {rep.t_solve_ms:.1f} ms ({rep.t_solve_ms / max(rep.iters, 1):.3f} ms/it) "
              f"err {err:.1e}", flush=True)
        op.close(); del x, b, xs; torch.cuda.empty_cache()
