timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py -q -x -p no:cacheprovider 2>&1 | tail -2
export CELLS="1,8 4,7 8,3 8,7 16,3 32,2"
for i in 1 2; do for v in old new; do echo "== $v"; SB_LIB=ab/$v.so timeout 900 python scripts/ab_dbg.py 0 2>&1 | tail -6; done; done
echo "== new, attention key splits auto"; SB_LIB=ab/new.so ATTN_SPLITS=0 timeout 900 python scripts/ab_dbg.py 0 2>&1 | tail -6
timeout 900 python scripts/iter_time_modes.py 2>&1 | tail -3
