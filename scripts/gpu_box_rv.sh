mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -x -m gpu -k "box_kernel_variants or block_apply_parity or full_size or essential or slabs or host_apply or tiny or setup_objects" 2>&1 | tail -5
timeout 600 python scripts/box_rv_time.py 4 2 3 5 6 2>&1
