nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r2s3a.json 2> gpurun_out/bench_r2s3a.err
tail -c 1500 gpurun_out/bench_r2s3a.json
