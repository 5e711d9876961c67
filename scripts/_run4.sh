timeout 600 python scripts/cta_trace.py 8 3 --pre 1 --json gpurun_out/cta_pre1.json > gpurun_out/cta_pre1.txt 2>&1
timeout 600 python scripts/cta_trace.py 8 3 --nopdl --json gpurun_out/cta_nopdl.json > gpurun_out/cta_nopdl.txt 2>&1
tail -8 gpurun_out/cta_pre1.txt; tail -8 gpurun_out/cta_nopdl.txt
