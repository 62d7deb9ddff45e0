# round-2 end evidence: full GPU suite, smoke, default bench line, launch list of the timed
# command, ncu --set full of the top kernel (roofline traffic), sanitizer memcheck on small cases
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -2 gpurun_out/bench_final.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --no-minres --e2e-steps 0 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:affine_apply -s 3 -c 1 -o /tmp/aff_final python scripts/ncu_target.py c4 4 5 > /dev/null 2>&1
ncu -i /tmp/aff_final.ncu-rep --page raw --csv > gpurun_out/raw_aff_final.csv 2>&1
python scripts/ncu_summary.py gpurun_out/raw_aff_final.csv > gpurun_out/ncu_aff_final.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/minres_kernels_final.csv python scripts/minres_kernels.py c4 4 chebyshev > /dev/null 2>&1
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize_cases.py c12 > gpurun_out/san_${t}_c12.log 2>&1; tail -2 gpurun_out/san_${t}_c12.log
done
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_cases.py tri > gpurun_out/san_memcheck_tri.log 2>&1; tail -2 gpurun_out/san_memcheck_tri.log
ls -la gpurun_out | tail -20
