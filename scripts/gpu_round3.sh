#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -8
python __graft_entry__.py smoke 2>&1 | tail -1
python scripts/tri_time.py 2>&1 | tail -12
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
