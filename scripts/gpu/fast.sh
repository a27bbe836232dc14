timeout 900 python -m pytest tests/test_gpu_full.py -m gpu -q --tb=short -k "grad_precision" > gpurun_out/gpu_fast.log 2>&1; grep -E "AssertionError|passed|failed" gpurun_out/gpu_fast.log | head
