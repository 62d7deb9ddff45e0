#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -q -x -k "variants or block_apply or full_size" 2>&1 | tail -3
bash scripts/halo_sweep.sh 2>&1 | grep -v Warn
ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:affine_apply -s 2 -c 1 python scripts/ncu_target.py c4 4 3 2>&1 | grep -E "affine|duration|wavefronts|conflicts|bytes" | head -12
