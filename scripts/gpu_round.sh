#!/bin/bash
# one gpurun session: tests, smoke, bench, ncu launch list + full capture of the top kernel
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -m pytest tests -m gpu -q -x 2>&1 | tail -15
python __graft_entry__.py smoke 2>&1 | tail -3
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --no-minres --e2e-steps 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:affine_apply -s 3 -c 1 -o gpurun_out/prof_affine_c4p4 python scripts/ncu_target.py c4 4 5 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
