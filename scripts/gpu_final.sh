#!/bin/bash
# end-of-round evidence: full GPU suite + smoke + default bench line (gpu_check.sh), then ncu of
# the trilinear batched kernel on config 3 and of the explicit W^-1 apply (winv target)
bash scripts/gpu_check.sh
PS="4" bash scripts/gpu_ncu_tri.sh > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:winv_apply -s 2 -c 1 -o /tmp/winv_p4 \
  python scripts/winv_target.py 4 > gpurun_out/ncu_winv.log 2>&1
ncu -i /tmp/winv_p4.ncu-rep --page raw --csv > gpurun_out/raw_winv_p4.csv 2>&1
python scripts/ncu_summary.py gpurun_out/raw_winv_p4.csv > gpurun_out/ncu_winv_p4.txt 2>&1
ls gpurun_out
