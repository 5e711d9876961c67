timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py -q -x -p no:cacheprovider 2>&1 | tail -2
for v in old new; do echo "== $v"; SB_LIB=ab/$v.so timeout 300 python scripts/cta_trace.py 8 127 --prefill > gpurun_out/pf_$v.txt 2>&1; head -1 gpurun_out/pf_$v.txt; done
export CELLS="8,7 16,8 32,2 32,8 64,2 64,8"
for v in old new; do echo "== $v"; SB_LIB=ab/$v.so timeout 900 python scripts/ab_dbg.py 0 2>&1 | tail -6; done
