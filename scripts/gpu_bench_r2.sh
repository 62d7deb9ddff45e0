# round-2 evidence run: default bench line + launch list of the timed command
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1200 python bench.py > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err; tail -3 gpurun_out/bench_r2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --no-minres --e2e-steps 0 > /dev/null 2>&1
ls -la gpurun_out/bench_r2.json gpurun_out/launches_r2.csv
