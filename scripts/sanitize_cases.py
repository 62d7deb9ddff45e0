"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck): configs 1 and 2
(block apply + MINRES with the Chebyshev and the AMG S^-1), box kernels p = 1..6 on ragged
meshes, the trilinear kernels (mass, gamma = 0 block, grad-div with explicit W^-1 and local CG),
essential sides, GMRES.  Run: compute-sanitizer --tool racecheck python scripts/sanitize_cases.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2304_12387_b200 import from_problem  # noqa: E402
from synth import make_config, random_vector  # noqa: E402


def run(pr, solve=True, **kw):
    op = from_problem(pr, **kw)
    n = op.sizes.n
    x = torch.from_numpy(random_vector(n, 3)).cuda()
    y = op.apply_block(x)
    op.apply_mass(x[:op.sizes.n_rt])
    if solve:
        op.minres(y, rtol=1e-10, maxit=40)
    torch.cuda.synchronize()
    op.close()


which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "c12"):
    run(make_config("c1"))
    run(make_config("c1"), schur="amg")
    run(make_config("c2"))
    run(make_config("c2"), schur="amg")
if which in ("all", "a9d"):   # reading A9d: Chebyshev polynomial in (V-cycle) S~, 3D and 2D
    run(make_config("c3", N=(4, 4, 3), p=2), schur="amg", amg_cheb_degree=3, amg_max_coarse=16)
    run(make_config("c3s", N=(3, 4, 3), p=2), schur="amg", amg_cheb_degree=2, amg_max_coarse=16)
    run(make_config("c1", N=(6, 5)), schur="amg", amg_cheb_degree=3, amg_max_coarse=8)
if which in ("all", "box"):
    for p, N in [(1, (9, 5, 5)), (2, (9, 5, 5)), (3, (5, 5, 3)), (4, (5, 3, 3)), (5, (4, 3, 3)),
                 (6, (4, 3, 2))]:
        pr = make_config("c2", N=N, p=p)
        pr.alpha = 10.0 ** random_vector(pr.E, 31)
        run(pr, solve=False)
    pr = make_config("c3s", N=(4, 4, 4), p=2)
    pr.affine = True
    pr.vertices = make_config("c2", N=(4, 4, 4), p=2).vertices
    run(pr, schur="amg")
if which in ("all", "tri"):
    for p in (1, 2, 3, 4, 5, 6):
        run(make_config("c3", N=(3, 2, 2), p=p), solve=(p <= 3))
        pr = make_config("c3", N=(2, 2, 3), p=p)
        pr.kind = "grad_div"
        pr.alpha = 10.0 ** random_vector(pr.E, 33)
        pr.beta = 10.0 ** random_vector(pr.E, 34)
        run(pr, solve=(p <= 3))
    pr = make_config("c3", N=(3, 3, 3), p=2)
    op = from_problem(pr, schur="amg")
    b = op.apply_block(torch.from_numpy(random_vector(op.sizes.n, 5)).cuda())
    op.gmres(b, rtol=1e-10, maxit=40, restart=10)
    torch.cuda.synchronize()
    op.close()
print("sanitize cases done", which)
