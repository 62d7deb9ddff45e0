#!/bin/bash
# variant parity + sweep (development aid)
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "variants" 2>&1 | tail -2
timeout 900 python scripts/variant_sweep.py $SWEEP_PS 2>&1 | grep -v Warn
