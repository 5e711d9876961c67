timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t9.txt 2>&1; tail -3 gpurun_out/t9.txt
timeout 600 python scripts/cta_trace.py 8 3 1 8 16 8 --json gpurun_out/cta_d.json > gpurun_out/cta_d.txt 2>&1; grep -A7 "per-layer" gpurun_out/cta_d.txt
