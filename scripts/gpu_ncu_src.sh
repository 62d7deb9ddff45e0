#!/bin/bash
# one ncu --set full capture (with source) of the affine block-apply kernel; source pages as CSV
for p in ${PS:-4 6}; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:affine_apply -s 2 -c 1 \
  -o /tmp/affine_p${p}_src python scripts/ncu_target.py c4 $p 3 > gpurun_out/ncu_p${p}.log 2>&1
ncu -i /tmp/affine_p${p}_src.ncu-rep --page source --csv --print-source cuda > gpurun_out/src_cuda_p${p}.csv 2>&1
ncu -i /tmp/affine_p${p}_src.ncu-rep --page source --csv --print-source sass > gpurun_out/src_sass_p${p}.csv 2>&1
ncu -i /tmp/affine_p${p}_src.ncu-rep --page raw --csv > gpurun_out/raw_p${p}.csv 2>&1
gzip -f gpurun_out/src_sass_p${p}.csv
done
ls -la gpurun_out
