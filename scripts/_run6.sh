timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t6.txt 2>&1
tail -3 gpurun_out/t6.txt
timeout 600 python scripts/cta_trace.py 8 3 1 8 --json gpurun_out/cta_vec.json > gpurun_out/cta_vec.txt 2>&1; grep -A7 "per-layer" gpurun_out/cta_vec.txt
