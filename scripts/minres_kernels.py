"""Per-kernel breakdown of MINRES iterations (development aid, run under ncu):
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
        python scripts/minres_kernels.py c4 4 amg
builds the operator, runs one warm-up solve (graph build) and one 6-iteration solve."""
import sys
sys.path.insert(0, ".")
import torch
from synth import make_config
from paper_2304_12387_b200 import from_problem

cfg, p, schur = sys.argv[1], int(sys.argv[2]), sys.argv[3]
pr = make_config(cfg, p=p)
op = from_problem(pr, schur=schur)
b = op.apply_block(torch.rand(op.sizes.n, dtype=torch.float64, device="cuda"))
op.minres(b, rtol=1e-30, maxit=6)
torch.cuda.synchronize()
print("MARK", flush=True)
op.minres(b, rtol=1e-30, maxit=6)
torch.cuda.synchronize()
