"""Box-kernel block apply at the bench sweep sizes (development aid; bench.py is the contract).
   python scripts/box_time.py [p ...]"""
import sys
import torch
sys.path.insert(0, ".")
from synth import make_config
from paper_2304_12387_b200 import from_problem
for p in [int(a) for a in (sys.argv[1:] or ["4", "2", "3", "5", "6"])]:
    N = {1: 192, 2: 160, 3: 128, 4: 128, 5: 96, 6: 80}[p]
    pr = make_config("c4", N=(N,) * 3, p=p)
    op = from_problem(pr, schur="chebyshev")
    n = op.sizes.n
    x = torch.rand(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for _ in range(5):
        op.apply_block(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(30):
        op.apply_block(x, y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 30
    b = 16 * n + 32 * pr.E
    print(f"p={p} N={N} {ms:.3f} ms {n / ms / 1e6:.1f} GDOF/s {b / ms / 1e6 / 6550.7 * 100:.1f}% HBM", flush=True)
    op.close()
    del x, y
    torch.cuda.empty_cache()
