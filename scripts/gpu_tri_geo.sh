mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "stored_geometry or multi_element or winv_modes or block_apply_parity or full_size" 2>&1 | tail -5
timeout 600 python scripts/tri_geo_time.py 4 2 3 5 6 2>&1 | tail -12
