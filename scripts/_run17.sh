timeout 600 python -m pytest tests/test_gpu_gqa_shapes.py tests/test_gpu_prefill_attention.py tests/test_gpu_model.py -q -x -p no:cacheprovider 2>&1 | tail -2
bash scripts/_run12.sh > gpurun_out/ab17.txt 2>&1; cat gpurun_out/ab17.txt
