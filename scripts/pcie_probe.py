"""dev: pinned host <-> device copy bandwidth (one direction at a time and both concurrently on
two streams) for the e2e ceiling: 4.3 GB each way, as config 4's x and y."""
import torch
n = 537657344
h_x = torch.empty(n, dtype=torch.float64).pin_memory()
h_y = torch.empty(n, dtype=torch.float64).pin_memory()
d_x = torch.empty(n, dtype=torch.float64, device="cuda")
d_y = torch.zeros(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
def h2d(): d_x.copy_(h_x, non_blocking=True)
def d2h(): h_y.copy_(d_y, non_blocking=True)
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d_x.copy_(h_x, non_blocking=True)
    with torch.cuda.stream(s2): h_y.copy_(d_y, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
gb = n * 8 / 1e9
for name, fn in [("h2d", h2d), ("d2h", d2h), ("both", both)]:
    ms = t(fn)
    print(f"{name}: {ms:.1f} ms, {gb / ms * 1e3:.1f} GB/s per direction", flush=True)
