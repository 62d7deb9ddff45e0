#!/bin/bash
python scripts/variant_sweep.py 2>&1 | grep -v Warn
for v in 4 10; do
HDIV_AFFINE_TILE=$v ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts.sum,sm__cycles_elapsed.avg --clock-control none -k regex:affine_apply -s 2 -c 1 python scripts/ncu_target.py c4 4 3 2>&1 | grep -E "duration|wavefronts|cycles" 
done
python -m pytest tests/test_gpu_parity.py -q -x -k "block_apply" 2>&1 | tail -1
