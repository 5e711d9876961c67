set -x
timeout 600 python -m pytest tests/test_gpu_tp.py -x -q -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/r2s3_tp.txt
timeout 900 python scripts/cta_trace.py 8 3 1 8 16 8 32 8 --json gpurun_out/cta_trace_r2.json > gpurun_out/cta_trace_r2.txt 2>&1
cat gpurun_out/r2s3_tp.txt
