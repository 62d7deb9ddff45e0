"""MINRES iteration count vs the number of z-slab ranks (reading A9c block-Jacobi AMG, with and
without the A9d polynomial, with and without the A9e global coarse space), on ONE GPU through the loopback communicator (iteration counts
only — no timing: loopback ranks share one device and meet at host barriers).
    python scripts/slab_iterations.py [N] [p] [P list, e.g. 1,2,4,8,16]"""
import sys
import threading
sys.path.insert(0, ".")
import numpy as np
import torch
from synth import make_config, random_vector
from paper_2304_12387_b200 import HdivOperator, from_problem, slabs
from paper_2304_12387_b200.binding import loopback_id

N = int(sys.argv[1]) if len(sys.argv) > 1 else 24
p = int(sys.argv[2]) if len(sys.argv) > 2 else 4
PS = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 2, 4, 8]
pr = make_config("c3", N=(N, N, N), p=p)
op = from_problem(pr, schur="amg", amg_cheb_degree=1)
b = op.apply_block(torch.from_numpy(random_vector(op.sizes.n, 3)).cuda()).cpu().numpy()
n_rt = op.sizes.n_rt
op.close()


def run(P, k, gc):
    if P == 1:
        o = from_problem(pr, schur="amg", amg_cheb_degree=k)
        _, rep = o.minres(torch.from_numpy(b).cuda(), rtol=1e-12, maxit=5000)
        o.close()
        return rep.iters, rep.converged
    uid = loopback_id(7000 + 100 * gc + 10 * P + k)
    out, errs = [None] * P, []

    def work(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                z0, z1 = slabs.slab_bounds(N, P, r)
                V, a, bb, g, e = slabs.slab_inputs(pr, z0, z1)
                o = HdivOperator(3, pr.N, p, pr.kind, vertices=V, alpha=a, beta=bb, gamma=g, eps=e,
                                 schur="amg", amg_cheb_degree=k, amg_global_coarse=1 if gc else 2,
                                 slab=(z0, z1), nccl_id=uid,
                                 rank=r, nranks=P)
                rt = slabs.local_to_global_rt(3, pr.N, p, z0, z1)
                l2 = slabs.local_to_global_l2(3, pr.N, p, z0, z1)
                bl = np.concatenate([b[:n_rt][rt], b[n_rt:][l2]])
                _, rep = o.minres(torch.from_numpy(bl).cuda(), rtol=1e-12, maxit=5000)
                out[r] = (rep.iters, rep.converged)
                torch.cuda.current_stream().synchronize()
                o.close()
        except Exception as ex:
            errs.append(ex)

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    return out[0]


print(f"config 3 mesh {N}^3, p = {p}, {len(b)} DOFs, b = A x*, rtol 1e-12", flush=True)
for gc in (0, 1):
    for k in (1, 3):
        for P in PS:
            if gc and P == 1:
                continue
            its, conv = run(P, k, gc)
            print(f"  A9d degree {k}, A9e global coarse {gc}, {P} slab ranks: {its} iterations "
                  f"(converged {bool(conv)})", flush=True)
