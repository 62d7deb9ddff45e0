"""Box-kernel block apply, sweep sizes: halo-tile kernel (HDIV_BOX_RV=0) vs rendezvous kernel.
Development aid; bench.py is the contract.   python scripts/box_rv_time.py [p ...]"""
import os, subprocess, sys
if len(sys.argv) > 1 and sys.argv[1] == "--one":
    import torch
    sys.path.insert(0, ".")
    from synth import make_config
    from paper_2304_12387_b200 import from_problem
    p = int(sys.argv[2])
    N = {1: 192, 2: 160, 3: 128, 4: 128, 5: 96, 6: 80}[p]
    pr = make_config("c4", N=(N,) * 3, p=p)
    op = from_problem(pr)
    n = op.sizes.n
    x = torch.rand(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for _ in range(5):
        op.apply_block(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(30):
        op.apply_block(x, y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 30
    b = 16 * n + 32 * pr.E
    print(f"p={p} N={N} rv={os.environ.get('HDIV_BOX_RV', '1')} {ms:.3f} ms {n / ms / 1e6:.1f} GDOF/s "
          f"{b / ms / 1e6 / 6550.7 * 100:.1f}% HBM", flush=True)
    sys.exit(0)
for p in (sys.argv[1:] or ["4", "2", "3", "5", "6"]):
    for rv in ("0", "1"):
        subprocess.run([sys.executable, __file__, "--one", p], env={**os.environ, "HDIV_BOX_RV": rv})
