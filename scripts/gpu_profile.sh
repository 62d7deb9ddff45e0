#!/bin/bash
# profiles/ evidence for a round: default bench line, the launch list of the same command
# (ncu gpu__time_duration, --clock-control none), one ncu --set full capture of the top kernel
# summarised here (the .ncu-rep stays on the box).  Usage: TAG=v11 bash scripts/gpu_profile.sh
set -u
TAG=${TAG:-vX}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -2 gpurun_out/bench_$TAG.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --no-minres --e2e-steps 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:affine_apply -s 3 -c 1 \
  -o /tmp/prof_affine_c4p4 python scripts/ncu_target.py c4 4 5 > /dev/null 2>&1
ncu -i /tmp/prof_affine_c4p4.ncu-rep --page raw --csv > gpurun_out/raw_affine_$TAG.csv 2>&1
python scripts/ncu_summary.py gpurun_out/raw_affine_$TAG.csv > gpurun_out/ncu_affine_c4p4_$TAG.txt 2>&1
ncu -i /tmp/prof_affine_c4p4.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/sass_affine_$TAG.csv.gz
ls -la gpurun_out
