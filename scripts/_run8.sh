timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py tests/test_gpu_headline_shapes.py tests/test_gpu_opt.py tests/test_gpu_gqa_shapes.py -x -q -p no:cacheprovider > gpurun_out/t8.txt 2>&1; tail -3 gpurun_out/t8.txt
timeout 600 python scripts/ab_dbg.py 0 16 > gpurun_out/ab_bulk.txt 2>&1; cat gpurun_out/ab_bulk.txt
