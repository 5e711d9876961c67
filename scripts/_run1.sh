set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/r2s3_gputest.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2s3_bench.json 2> gpurun_out/r2s3_bench.err
tail -3 gpurun_out/r2s3_gputest.txt; tail -c 600 gpurun_out/r2s3_bench.json
