#!/bin/bash
# r02 probe: DMMA vs DFMA peak, source-level ncu of the box kernel (p=4, 6) and trilinear p=4
mkdir -p gpurun_out
./scripts/dmma_peak > gpurun_out/dmma_peak.txt 2>&1
./scripts/fp64_peak >> gpurun_out/dmma_peak.txt 2>&1
PS="4 6" bash scripts/gpu_ncu_src.sh > /dev/null 2>&1
for p in 4 6; do python scripts/sass_hot.py gpurun_out/src_sass_p${p}.csv.gz > gpurun_out/sass_hot_p${p}.txt 2>&1; python scripts/ncu_summary.py gpurun_out/raw_p${p}.csv >> gpurun_out/sass_hot_p${p}.txt 2>&1; done
PS="4" bash scripts/gpu_ncu_tri.sh > /dev/null 2>&1
ls -la gpurun_out
