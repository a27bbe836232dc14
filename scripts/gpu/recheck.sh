# Re-entry check: full GPU suite + default bench line.
timeout 1500 python -m pytest tests -m gpu -q --tb=short -x > gpurun_out/gpu_full.log 2>&1; tail -3 gpurun_out/gpu_full.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 1500 gpurun_out/bench_default.json
