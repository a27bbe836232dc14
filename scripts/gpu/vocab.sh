timeout 900 python -m pytest tests/test_gpu_full.py -m gpu -q -x --tb=short -k "vocab_sharded" > gpurun_out/gpu_vocab.log 2>&1; tail -15 gpurun_out/gpu_vocab.log
