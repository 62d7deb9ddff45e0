"""Box-kernel tile-variant sweep at the bench sizes (development aid).  One operator per order;
HDIV_AFFINE_TILE is re-read by the library at every launch, so variants switch in-process.
    python scripts/variant_sweep.py [p ...]"""
import os, sys
sys.path.insert(0, ".")
import torch
from synth import make_config
from paper_2304_12387_b200 import from_problem

SIZES = {2: 160, 3: 128, 4: 128, 5: 96, 6: 80}
VARS = {2: [0], 3: [7], 4: [4], 5: [12, 10], 6: [12, 10]}
ps = [int(a) for a in sys.argv[1:]] or [2, 3, 4, 5, 6]
os.environ["HDIV_MARCH_TILE"] = "-1"
for p in ps:
    N = SIZES[p]
    op = from_problem(make_config("c4", N=(N, N, N), p=p))
    n = op.sizes.n
    x = torch.rand(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    res = {v: [] for v in VARS[p]}
    for rep in range(3):
        for v in VARS[p]:
            os.environ["HDIV_AFFINE_TILE"] = str(v)
            for _ in range(3):
                op.apply_block(x, y)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(20):
                op.apply_block(x, y)
            e1.record()
            torch.cuda.synchronize()
            res[v].append(e0.elapsed_time(e1) / 20)
    for v, t in res.items():
        ms = min(t)
        print(f"p={p} N={N} variant {v}: best {ms:.3f} ms (runs {', '.join(f'{a:.3f}' for a in t)}) "
              f"{n / ms / 1e6:.1f} GDOF/s {16 * n / ms / 1e6 / 6534.8 * 100:.1f}% HBM", flush=True)
    op.close()
    del x, y
    torch.cuda.empty_cache()
