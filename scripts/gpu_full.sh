# full GPU suite + MINRES / AMG / GMRES timings (development check)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python scripts/minres_time.py 2>&1
timeout 600 python scripts/amg_time.py 2>&1 | tail -8
timeout 600 python scripts/gmres_time.py 2>&1 | tail -4
