mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -x -m gpu -k "preconditioner or minres or amg or slabs or essential or gamma or gmres or config2" 2>&1 | tail -2
timeout 600 python scripts/minres_time.py 2>&1 | head -2
timeout 600 python scripts/amg_time.py 2>&1 | grep "c4\|c3"
