import os, sys
sys.path.insert(0, ".")
import torch
from synth import make_config, random_vector
from paper_2304_12387_b200 import from_problem
def t(fn, iters=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters
for p in (2, 3, 4, 5, 6):
    pr = make_config("c3", N=(48, 48, 48), p=p)
    pr.kind = "grad_div"; pr.alpha = 10.0 ** random_vector(pr.E, 33); pr.beta = 10.0 ** random_vector(pr.E, 34)
    op = from_problem(pr)
    x = torch.rand(op.sizes.n, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
    q = x[op.sizes.n_rt:].clone(); yq = torch.empty_like(q)
    print(f"p={p} grad-div jittered 48^3: block {t(lambda: op.apply_block(x, y)):.3f} ms  Z {t(lambda: op.apply_z(q, yq)):.3f} ms", flush=True)
    op.close(); torch.cuda.empty_cache()
