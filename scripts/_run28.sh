timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 900 python scripts/iter_time_modes.py 2>&1 | tail -3
