"""dev (ncu target): a few A9e MINRES iterations on 2 loopback slab ranks of the config-3 mesh."""
import sys
import threading
sys.path.insert(0, ".")
import numpy as np
import torch
from synth import make_config, random_vector
from paper_2304_12387_b200 import HdivOperator, slabs
from paper_2304_12387_b200.binding import loopback_id
N = int(sys.argv[1]) if len(sys.argv) > 1 else 48
P = 2
pr = make_config("c3", N=(N, N, N), p=4)
uid = loopback_id(9001)


def work(r):
    torch.cuda.set_device(0)
    with torch.cuda.stream(torch.cuda.Stream()):
        z0, z1 = slabs.slab_bounds(N, P, r)
        V, a, bb, g, e = slabs.slab_inputs(pr, z0, z1)
        o = HdivOperator(3, pr.N, 4, pr.kind, vertices=V, alpha=a, beta=bb, gamma=g, eps=e,
                         schur="amg", amg_cheb_degree=3, amg_global_coarse=1, slab=(z0, z1),
                         nccl_id=uid, rank=r, nranks=P)
        b = torch.from_numpy(random_vector(o.sizes.n, 1 + r)).cuda()
        o.minres(b, rtol=1e-30, maxit=6)
        torch.cuda.current_stream().synchronize()
        o.close()


th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
for t in th:
    t.start()
for t in th:
    t.join()
print("done")
