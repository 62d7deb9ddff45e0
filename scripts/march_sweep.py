"""Sweep z-chunk length / tile variants of the z-marching box kernel (env vars are read per launch)."""
import os, sys
sys.path.insert(0, ".")
import torch
from synth import make_config
from paper_2304_12387_b200 import from_problem

def t(op, x, y, n=20):
    for _ in range(3): op.apply_block(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): op.apply_block(x, y)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n

for p, N in [(4, 128), (2, 160), (3, 128), (5, 96), (6, 80)]:
    pr = make_config("c4", N=(N, N, N), p=p)
    op = from_problem(pr)
    x = torch.rand(op.sizes.n, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
    n = op.sizes.n
    res = []
    for mv in ("0", "1", "-1"):
        for zc in (["4", "8", "16", "32"] if mv != "-1" else ["0"]):
            os.environ["HDIV_MARCH_TILE"] = mv
            if zc == "0": os.environ.pop("HDIV_ZCHUNK", None)
            else: os.environ["HDIV_ZCHUNK"] = zc
            ms = t(op, x, y)
            res.append((ms, mv, zc))
            print(f"p={p} march={mv:>2} zchunk={zc:>2}: {ms:.3f} ms {16*n/ms/1e6/6534.8*100:.1f}% HBM", flush=True)
    best = min(res)
    print(f"BEST p={p}: {best}", flush=True)
    op.close(); del x, y; torch.cuda.empty_cache()
os.environ.pop("HDIV_ZCHUNK", None); os.environ.pop("HDIV_MARCH_TILE", None)
exec(open("scripts/quick_time.py").read().split("for p in")[0])
run("c3", 4); run("c3", 2, (96, 96, 96)); run("c3", 6, (48, 48, 48))
