"""e2e (pinned host -> device -> host) block apply vs HDIV_HOST_CHUNKS (dev aid)."""
import os, sys, time
sys.path.insert(0, ".")
import torch
from synth import make_config
from paper_2304_12387_b200 import from_problem
op = from_problem(make_config("c4"))
n = op.sizes.n
xh = torch.rand(n, dtype=torch.float64).pin_memory()
yh = torch.empty(n, dtype=torch.float64).pin_memory()
for ch in sys.argv[1:] or ["16", "32", "64"]:
    os.environ["HDIV_HOST_CHUNKS"] = ch
    for _ in range(2):
        op.apply_block_host(xh, yh)
    t0 = time.perf_counter()
    for _ in range(5):
        op.apply_block_host(xh, yh)
    t = (time.perf_counter() - t0) / 5
    print(f"chunks {ch}: {t * 1e3:.1f} ms per e2e apply, {n / t / 1e9:.2f} GDOF/s", flush=True)
