#!/bin/bash
# ncu --set full (with SASS source) of the trilinear block apply on config 3 (p = 2, 3, 4)
for p in ${PS:-4}; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tri_ -s 2 -c 1 \
  -o /tmp/tri_p${p} python scripts/ncu_target.py c3 $p 3 > gpurun_out/ncu_tri_p${p}.log 2>&1
ncu -i /tmp/tri_p${p}.ncu-rep --page raw --csv > gpurun_out/raw_tri_p${p}.csv 2>&1
ncu -i /tmp/tri_p${p}.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/src_sass_tri_p${p}.csv.gz
python scripts/ncu_summary.py gpurun_out/raw_tri_p${p}.csv > gpurun_out/ncu_tri_p${p}.txt 2>&1
python scripts/sass_hot.py gpurun_out/src_sass_tri_p${p}.csv.gz >> gpurun_out/ncu_tri_p${p}.txt 2>&1
done
ls -la gpurun_out
