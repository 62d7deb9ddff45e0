mkdir -p gpurun_out
for e in 1 2; do echo "== EPC $e"; HDIV_TRI_EPC=$e timeout 300 python scripts/tri_geo_time.py 4 3 2>&1 | tail -4; done
# stored-G trilinear kernel, config 3 p=4 (block apply, gamma = 0)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tri_multi -s 2 -c 1 -o /tmp/tri_sg python scripts/ncu_target.py c3 4 3 > gpurun_out/ncu_tri_sg.log 2>&1
ncu -i /tmp/tri_sg.ncu-rep --page raw --csv > gpurun_out/raw_tri_sg.csv 2>&1
ncu -i /tmp/tri_sg.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/src_sass_tri_sg.csv.gz
python scripts/ncu_summary.py gpurun_out/raw_tri_sg.csv > gpurun_out/ncu_tri_sg.txt 2>&1
python scripts/sass_hot.py gpurun_out/src_sass_tri_sg.csv.gz >> gpurun_out/ncu_tri_sg.txt 2>&1
# W^-1: explicit inverses (p=4) and the local CG (p=4, 6)
timeout 600 ncu --set full --clock-control none -k regex:winv_apply -s 2 -c 1 -o /tmp/winv_p4 python scripts/winv_target.py 4 > gpurun_out/ncu_winv.log 2>&1
ncu -i /tmp/winv_p4.ncu-rep --page raw --csv > gpurun_out/raw_winv_p4.csv 2>&1
python scripts/ncu_summary.py gpurun_out/raw_winv_p4.csv > gpurun_out/ncu_winv_p4.txt 2>&1
for p in 4 6; do
HDIV_WINV=cg timeout 600 ncu --set full --clock-control none -k regex:tri_kernel -s 2 -c 1 -o /tmp/wcg_p$p python scripts/winv_target.py $p > gpurun_out/ncu_wcg_p$p.log 2>&1
ncu -i /tmp/wcg_p$p.ncu-rep --page raw --csv > gpurun_out/raw_wcg_p$p.csv 2>&1
python scripts/ncu_summary.py gpurun_out/raw_wcg_p$p.csv > gpurun_out/ncu_wcg_p$p.txt 2>&1
done
ls gpurun_out | head -50
