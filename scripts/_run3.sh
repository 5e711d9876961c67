timeout 900 python scripts/pdl_knobs.py > gpurun_out/pdl_knobs.txt 2>&1
timeout 900 python scripts/cta_trace.py 8 3 1 8 16 8 --json gpurun_out/cta_trace_r2b.json > gpurun_out/cta_trace_r2b.txt 2>&1
cat gpurun_out/pdl_knobs.txt
