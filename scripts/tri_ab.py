"""dev: config-3 block apply time (stored G and on-the-fly J) for A/B."""
import sys
sys.path.insert(0, ".")
import torch
from synth import make_config
from paper_2304_12387_b200 import from_problem
for geo in (2, 1):
    op = from_problem(make_config("c3"), tri_geometry=geo, schur="chebyshev")
    x = torch.rand(op.sizes.n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        op.apply_block(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(30):
        op.apply_block(x, y)
    e1.record()
    torch.cuda.synchronize()
    print(f"tri_geometry {geo}: {e0.elapsed_time(e1) / 30:.3f} ms", flush=True)
    op.close()
