mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -x -m gpu -k "box_kernel_variants or (block_apply_parity and (c2 or c5)) or essential or slabs or tiny" 2>&1 | tail -2
echo "== dmma Mh"; timeout 300 python scripts/box_time.py 5 6 2>&1
