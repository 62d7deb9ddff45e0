#!/bin/bash
# Dev aid: build libhdiv variants that differ only in kernel_affine.cu compile-time switches,
# into gpurun_variants/libhdiv_<name>.so (A/B timing on the GPU box: copy one over
# paper_2304_12387_b200/libhdiv.so, run bench.py).  Usage: scripts/affine_variants.sh name "-DFLAG=.." ...
# VSRC=solver.cu (default kernel_affine.cu): the source file the flags apply to.
set -e
cd "$(dirname "$0")/.."
python -m paper_2304_12387_b200.build > /dev/null
mkdir -p gpurun_variants
OBJ=paper_2304_12387_b200/build_obj
while [ $# -gt 0 ]; do
  name=$1; flags=$2; shift 2
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -O3 \
    --expt-relaxed-constexpr -diag-suppress 177 -Iinclude -Ipaper_2304_12387_b200/csrc $flags \
    -c paper_2304_12387_b200/csrc/${VSRC:-kernel_affine.cu} -o /tmp/ka_$name.o &
  pids="$pids $!"; names="$names $name"
done
wait $pids
for name in $names; do
  objs=""
  for s in tables.cpp kernel_affine.cu kernel_general.cu kernel_trilinear.cu kernel_sparse.cu amg.cu gmres.cu solver.cu comm.cu api.cu; do
    [ "$s" = "${VSRC:-kernel_affine.cu}" ] || objs="$objs $OBJ/$s.o"
  done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o gpurun_variants/libhdiv_$name.so /tmp/ka_$name.o $objs -ldl -cudart static
  echo gpurun_variants/libhdiv_$name.so
done
