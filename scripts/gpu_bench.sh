#!/bin/bash
# full bench + launch list + ncu capture of the top kernel (profiles/ evidence)
mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -2
python __graft_entry__.py smoke 2>&1 | tail -1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --no-minres --e2e-steps 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:affine_apply -s 3 -c 1 -o gpurun_out/prof_affine_c4p4_bench python scripts/ncu_target.py c4 4 5 > /dev/null 2>&1
ls gpurun_out
