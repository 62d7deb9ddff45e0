mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -x -m gpu -k "preconditioner or minres or slabs or essential or gamma or config2 or gmres" 2>&1 | tail -3
echo "== cells m8u1"; timeout 600 python scripts/minres_time.py 2>&1
timeout 300 python scripts/gmres_time.py 2>&1 | tail -5
