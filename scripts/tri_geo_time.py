"""Trilinear block / mass apply on config 3 (and the sweep orders on the 64^3 / 48^3 jittered
meshes): on-the-fly Jacobian (tri_geometry=1) vs stored quadrature-point factors (=2).
Development aid; bench.py is the contract."""
import sys
import torch
sys.path.insert(0, ".")
from synth import make_config, random_vector
from paper_2304_12387_b200 import from_problem


def t(op, x, y, n=20, mass=False):
    f = (lambda: op.apply_mass(x, y)) if mass else (lambda: op.apply_block(x, y))
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for p in [int(a) for a in (sys.argv[1:] or ["4", "2", "3", "5", "6"])]:
    N = (64, 64, 64) if p <= 4 else (48, 48, 48)
    for gd in (False, True):
        pr = make_config("c3", N=N, p=p)
        if gd:
            pr.kind = "grad_div"
            pr.alpha = 10.0 ** random_vector(pr.E, 33, -2.0, 2.0)
            pr.beta = 10.0 ** random_vector(pr.E, 34, -2.0, 2.0)
        res = []
        for g in (1, 2):
            try:
                op = from_problem(pr, tri_geometry=g)
            except Exception as ex:
                res.append(f"geo{g}: {ex}")
                continue
            x = torch.rand(op.sizes.n, dtype=torch.float64, device="cuda")
            y = torch.empty_like(x)
            ms = t(op, x, y)
            u = x[:op.sizes.n_rt].contiguous()
            yu = torch.empty_like(u)
            msm = t(op, u, yu, mass=True)
            res.append(f"geo{g}: block {ms:.3f} ms ({op.sizes.n / ms / 1e6:.1f} GDOF/s) mass {msm:.3f} ms")
            op.close()
            del x, y, u, yu
            torch.cuda.empty_cache()
        print(f"p={p} N={N[0]} {'graddiv' if gd else 'darcy-g0'}: " + " | ".join(res), flush=True)
