"""A/B of the trilinear mass / gamma = 0 block apply: the one-element tri_kernel (HDIV_TRI_EPC=0) vs
EPC elements per 96-thread CTA (dev aid).  python scripts/tri_epc.py"""
import os
import sys
import torch
sys.path.insert(0, ".")
from synth import make_config
from paper_2304_12387_b200 import from_problem


def t(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


for p in [int(v) for v in (sys.argv[1:] or (1, 2, 3, 4, 5, 6))]:
    pr = make_config("c3", N=(64, 64, 64) if p < 6 else (48, 48, 48), p=p)
    op = from_problem(pr)
    n, nrt = op.sizes.n, op.sizes.n_rt
    x = torch.rand(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    ref = None
    for epc in ("0", "1", "2", "3", "4"):
        if (epc == "2" and p > 5) or (epc == "3" and p > 4) or (epc == "4" and p > 3):
            continue
        os.environ["HDIV_TRI_EPC"] = epc
        mb = t(lambda: op.apply_block(x, y))
        yb = y.clone()
        mm = t(lambda: op.apply_mass(x[:nrt], y[:nrt]))
        if ref is None:
            ref = yb
        d = ((yb - ref).abs().max() / ref.abs().max()).item()
        print(f"p={p} EPC={epc} block {mb:.3f} ms {n / mb / 1e6:.1f} GDOF/s | mass {mm:.3f} ms | rel diff vs EPC=0 {d:.1e}",
              flush=True)
    op.close()
    del x, y, ref, yb
    torch.cuda.empty_cache()
