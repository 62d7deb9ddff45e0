mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -x -m gpu -k "trilinear or (block_apply_parity and c3) or essential" 2>&1 | tail -2
timeout 300 python scripts/tri_geo_time.py 4 3 2>&1 | grep darcy
