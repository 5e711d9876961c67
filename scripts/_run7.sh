timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py tests/test_gpu_prefill_attention.py tests/test_gpu_gqa_shapes.py -x -q -p no:cacheprovider > gpurun_out/t7.txt 2>&1; tail -2 gpurun_out/t7.txt
timeout 600 python scripts/cta_trace.py 8 3 1 8 --json gpurun_out/cta_att.json > gpurun_out/cta_att.txt 2>&1; grep -A7 "per-layer" gpurun_out/cta_att.txt
timeout 600 python scripts/ab_dbg.py 0 > gpurun_out/ab_att.txt 2>&1; cat gpurun_out/ab_att.txt
