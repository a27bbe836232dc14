# NEXT-3 top-k baseline tests + LSE tests; bench lines of the modes
timeout 900 python -m pytest tests/test_gpu_topk.py tests/test_gpu_lse.py -q --tb=short > gpurun_out/gpu_topk.log 2>&1; tail -25 gpurun_out/gpu_topk.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --topk 32 > gpurun_out/bench_topk.json 2> gpurun_out/bench_topk.err; tail -c 300 gpurun_out/bench_topk.json; tail -3 gpurun_out/bench_topk.err
