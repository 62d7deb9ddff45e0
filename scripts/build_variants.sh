# dev: build libhdiv variants with extra kernel_affine.cu defines into gpurun_variants/
#   VARIANTS="name:-DFOO=1 -DBAR=2;name2:..." bash scripts/build_variants.sh
set -e
cd "$(dirname "$0")/.."
python -c "from paper_2304_12387_b200 import build as b; b.build()" > /dev/null
mkdir -p gpurun_variants
O=paper_2304_12387_b200/build_obj
NV=/usr/local/cuda/bin/nvcc
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="-O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr -diag-suppress 177 -Iinclude -Ipaper_2304_12387_b200/csrc"
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  n=${v%%:*}; f=${v#*:}
  ( $NV $ARCH $FL $f -c paper_2304_12387_b200/csrc/kernel_affine.cu -o /tmp/ka_$n.o && \
    objs=$(for s in tables.cpp kernel_general.cu kernel_trilinear.cu kernel_sparse.cu amg.cu gmres.cu solver.cu comm.cu api.cu; do echo $O/$s.o; done) && \
    $NV $ARCH -shared -o gpurun_variants/libhdiv_$n.so /tmp/ka_$n.o $objs -ldl -cudart static && echo "built $n" ) &
done
wait
