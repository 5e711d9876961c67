timeout 2400 python bench.py --workload trace > gpurun_out/bench_trace_r2c.json 2> gpurun_out/bench_trace_r2c.err; tail -c 2500 gpurun_out/bench_trace_r2c.json
