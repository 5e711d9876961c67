timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py tests/test_gpu_headline_shapes.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 300 python scripts/cta_trace.py 8 127 --prefill --json gpurun_out/cta_pf2.json > gpurun_out/cta_pf2.txt 2>&1; head -1 gpurun_out/cta_pf2.txt; grep -A7 "per-layer" gpurun_out/cta_pf2.txt | head -8
export CELLS="1,8 8,3 8,7 16,3 32,2 64,2"
for v in old new; do echo "== $v"; SB_LIB=ab/$v.so timeout 900 python scripts/ab_dbg.py 0 2>&1 | tail -6; done
