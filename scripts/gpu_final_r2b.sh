# round-2 (late) evidence: full GPU suite, smoke, default bench line, launch list of the timed
# command, ncu --set full of the top kernel, sanitizer on the A9d and box cases
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1500 python bench.py > gpurun_out/bench_r02_v4.json 2> gpurun_out/bench_r02_v4.err; tail -2 gpurun_out/bench_r02_v4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_v4.csv python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --no-minres --e2e-steps 0 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:affine_apply -s 3 -c 1 -o /tmp/aff_v4 python scripts/ncu_target.py c4 4 5 > /dev/null 2>&1
ncu -i /tmp/aff_v4.ncu-rep --page raw --csv > gpurun_out/raw_aff_v4.csv 2>&1
python scripts/ncu_summary.py gpurun_out/raw_aff_v4.csv > gpurun_out/ncu_aff_v4.txt 2>&1
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize_cases.py a9d > gpurun_out/san_${t}_a9d.log 2>&1; tail -2 gpurun_out/san_${t}_a9d.log
done
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_cases.py box > gpurun_out/san_racecheck_box_v4.log 2>&1; tail -2 gpurun_out/san_racecheck_box_v4.log
ls -la gpurun_out | tail -20
