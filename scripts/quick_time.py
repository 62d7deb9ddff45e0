"""Quick device timing of the block apply (development aid; bench.py is the contract)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from synth import make_config
from paper_2304_12387_b200 import from_problem

def run(name, p, N=None, iters=20):
    pr = make_config(name, N=N, p=p)
    t0 = time.time(); op = from_problem(pr); ts = time.time() - t0
    n = op.sizes.n
    x = torch.rand(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3): op.apply_block(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters): op.apply_block(x, y)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    gb = 16 * n / 1e9
    print(f"{name} p={p} N={pr.N} n={n} setup {ts:.1f}s  apply {ms:.3f} ms  {n/ms/1e6:.1f} GDOF/s  {gb/ms*1e3:.0f} GB/s ({gb/ms*1e3/6534.8*100:.1f}% of 6534.8)", flush=True)
    op.close(); del x, y; torch.cuda.empty_cache()

for p in [4, 2, 3, 5, 6]:
    N = {2: (160,)*3, 3: (128,)*3, 4: (128,)*3, 5: (96,)*3, 6: (80,)*3}[p]
    run("c4", p, N)
run("c3", 4)
