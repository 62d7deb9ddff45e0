"""Timing-variance diagnostic for the p=4 box apply (development aid)."""
import os, sys, subprocess
sys.path.insert(0, ".")
import torch
from synth import make_config
from paper_2304_12387_b200 import from_problem

def clocks():
    r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,clocks_throttle_reasons.active",
                        "--format=csv,noheader"], capture_output=True, text=True)
    return r.stdout.strip()

def timeit(op, x, y, it=50):
    for _ in range(3): op.apply_block(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(it): op.apply_block(x, y)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it

order = sys.argv[1:] or ["4", "0", "4", "6", "4"]
op = from_problem(make_config("c4", p=4))
n = op.sizes.n
x = torch.rand(n, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
for v in order:
    os.environ["HDIV_AFFINE_TILE"] = v
    ms = timeit(op, x, y)
    print(f"variant {v}: {ms:.3f} ms  {16*n/ms/1e6/6534.8*100:.1f}%  [{clocks()}]", flush=True)
# fresh buffers
x2 = torch.rand(n, dtype=torch.float64, device="cuda"); y2 = torch.empty_like(x2)
os.environ["HDIV_AFFINE_TILE"] = "4"
print(f"fresh buffers v4: {timeit(op, x2, y2):.3f} ms", flush=True)
print(f"old buffers v4: {timeit(op, x, y):.3f} ms", flush=True)
