# A/B of dev variants (gpurun_variants/libhdiv_<v>.so) on one box: minres / amg per-iteration time
mkdir -p gpurun_out
cp paper_2304_12387_b200/libhdiv.so /tmp/libhdiv_base.so
for v in base ${VARIANTS} base; do
  [ "$v" = base ] && cp /tmp/libhdiv_base.so paper_2304_12387_b200/libhdiv.so || cp gpurun_variants/libhdiv_$v.so paper_2304_12387_b200/libhdiv.so
  echo "== $v"; timeout 600 python ${SCRIPT:-scripts/minres_time.py} 2>&1 | ${FILTER:-head -2}
done
cp /tmp/libhdiv_base.so paper_2304_12387_b200/libhdiv.so
