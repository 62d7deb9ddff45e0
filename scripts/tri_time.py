"""Device timing of the trilinear block apply with and without the W^-1 local CG (dev aid)."""
import sys
import torch
sys.path.insert(0, ".")
from synth import make_config, random_vector
from paper_2304_12387_b200 import from_problem


def run(tag, p, N=(64, 64, 64), iters=10):
    pr = make_config("c3", N=N, p=p)
    if tag == "grad_div":
        pr.kind = "grad_div"
        pr.alpha = 10.0 ** random_vector(pr.E, 33)
        pr.beta = 10.0 ** random_vector(pr.E, 34)
    elif tag == "darcy_gamma":
        pr.gamma = 10.0 ** random_vector(pr.E, 35)
    op = from_problem(pr)
    n = op.sizes.n
    x = torch.rand(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        op.apply_block(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters):
        op.apply_block(x, y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    print(f"c3 {tag} p={p} N={N} n={n} apply {ms:.3f} ms  {n / ms / 1e6:.1f} GDOF/s", flush=True)
    op.close()
    torch.cuda.empty_cache()


for p in (2, 4, 6):
    for tag in ("darcy0", "darcy_gamma", "grad_div"):
        run(tag, p, N=(64, 64, 64) if p < 6 else (40, 40, 40))
