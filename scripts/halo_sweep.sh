#!/bin/bash
# halo-tile kernel variants (HDIV_MARCH_TILE=-1, HDIV_AFFINE_TILE=v), p = 2..6
for v in 0 1 2 4 5; do
  HDIV_MARCH_TILE=-1 HDIV_AFFINE_TILE=$v python - <<'PY'
import os, sys
sys.path.insert(0, ".")
import torch
from synth import make_config
from paper_2304_12387_b200 import from_problem
v = os.environ["HDIV_AFFINE_TILE"]
for p, N in [(2, 160), (3, 128), (4, 128), (5, 96), (6, 80)]:
    pr = make_config("c4", N=(N, N, N), p=p)
    op = from_problem(pr)
    x = torch.rand(op.sizes.n, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
    for _ in range(3): op.apply_block(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20): op.apply_block(x, y)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    n = op.sizes.n
    print(f"halo variant {v} p={p} N={N}: {ms:.3f} ms {n/ms/1e6:.1f} GDOF/s {16*n/ms/1e6/6534.8*100:.1f}% HBM", flush=True)
    op.close(); del x, y; torch.cuda.empty_cache()
PY
done
