"""paper_2304_12387_b200 — B200-native hot path of arXiv 2304.12387 (matrix-free block-
preconditioned MINRES for RT/L2 grad-div and Darcy saddle-point systems).

The compute lives in `libhdiv.so` (hand-written sm_100a CUDA behind the C-ABI of
`include/hdiv.h`); `binding` is a thin ctypes layer.  There is no CPU fallback.
"""
from .binding import (HdivOperator, HdivError, load_library, from_problem,  # noqa: F401
                      LIB_PATH, GRAD_DIV, DARCY)
