rm -f gpurun_out/parity.jsonl
KD_PARITY_LOG=$PWD/gpurun_out/parity.jsonl timeout 1500 python -m pytest tests -m gpu -q --tb=short > gpurun_out/gpu_full.log 2>&1; tail -3 gpurun_out/gpu_full.log; wc -l gpurun_out/parity.jsonl
