python -m pytest tests -q -m gpu -x -k "winv_modes or apply_z or c3g or trilinear or gamma or essential or multi_element" 2>&1 | tail -3
python scripts/tri_z_time.py
HDIV_WINV=cg python scripts/tri_z_time.py
python - <<'PY'
import json, sys, torch
sys.path.insert(0, ".")
import bench
print(json.dumps(bench.winv_bench(torch))[:1500])
PY
