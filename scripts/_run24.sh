SB_SKIP_CPU=1 timeout 1200 python bench.py --workload opt --steps 3 --warmup 3 > gpurun_out/bench_opt_r2c.json 2> gpurun_out/bench_opt_r2c.err; tail -c 800 gpurun_out/bench_opt_r2c.json
SB_SKIP_CPU=1 timeout 1500 python bench.py --workload 70b --steps 3 --warmup 3 > gpurun_out/bench_70b_r2c.json 2> gpurun_out/bench_70b_r2c.err; tail -c 800 gpurun_out/bench_70b_r2c.json
