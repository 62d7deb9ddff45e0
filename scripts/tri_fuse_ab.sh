#!/bin/bash
# A/B: explicit W^-1 fused into the batched trilinear kernel's y_q store vs a separate apply
python -m pytest tests -q -m gpu -x -k "winv_modes or c3g or multi_element or apply_z" 2>&1 | tail -2
HDIV_WINV_FUSE=0 python -m pytest tests -q -m gpu -x -k "winv_modes" 2>&1 | tail -1
echo FUSED; python scripts/tri_z_time.py
echo SEPARATE; HDIV_WINV_FUSE=0 python scripts/tri_z_time.py
