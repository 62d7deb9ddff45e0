#!/bin/bash
# A/B of the trilinear kernel CTA size (64 vs 96 threads) at p = 1..6
for nt in 64 96; do
  echo "NT=$nt"
  HDIV_TRI_NT=$nt timeout 300 python - <<'PY' 2>&1 | grep -v Warn
import sys, torch, numpy as np
sys.path.insert(0, ".")
from synth import make_config, random_vector
from paper_2304_12387_b200 import from_problem
for p in (1, 2, 3, 4, 5, 6):
    N = {1: 128, 2: 96, 3: 72, 4: 64, 5: 48, 6: 40}[p]
    for tag in ("darcy0", "grad_div"):
        pr = make_config("c3", N=(N, N, N), p=p)
        if tag == "grad_div":
            pr.kind, pr.alpha, pr.beta = "grad_div", 10.0 ** random_vector(pr.E, 33), 10.0 ** random_vector(pr.E, 34)
        op = from_problem(pr)
        x = torch.rand(op.sizes.n, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
        for _ in range(3): op.apply_block(x, y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(10): op.apply_block(x, y)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"  p={p} {tag:8s} {ms:.3f} ms {op.sizes.n / ms / 1e6:.1f} GDOF/s", flush=True)
        op.close(); del x, y; torch.cuda.empty_cache()
PY
done
