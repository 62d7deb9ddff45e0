#!/bin/bash
mkdir -p gpurun_out
for mv in 0 1; do
HDIV_MARCH_TILE=$mv python - <<'PY'
import os, sys
sys.path.insert(0, ".")
import torch
from synth import make_config
from paper_2304_12387_b200 import from_problem
for p, N in [(3, 128), (4, 128), (5, 96), (6, 80)]:
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
    print(f"march variant {os.environ['HDIV_MARCH_TILE']} p={p} N={N}: {ms:.3f} ms {n/ms/1e6:.1f} GDOF/s {16*n/ms/1e6/6534.8*100:.1f}% HBM", flush=True)
    op.close(); del x, y; torch.cuda.empty_cache()
PY
done
python scripts/quick_time.py 2>&1 | grep -v Warn
ncu --set full --clock-control none --import-source on -k regex:affine_apply -s 2 -c 1 -o gpurun_out/prof_affine_c4p4_v9 python scripts/ncu_target.py c4 4 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:affine_apply -s 2 -c 1 -o gpurun_out/prof_affine_c4p6_v1 python scripts/ncu_target.py c4 6 3 > /dev/null 2>&1
ls gpurun_out
