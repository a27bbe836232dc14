# Staged variant: parity tests + bench lines.
timeout 1200 python -m pytest tests/test_gpu_stage.py -q --tb=short -x > gpurun_out/stage_tests.log 2>&1; tail -15 gpurun_out/stage_tests.log
timeout 600 python bench.py --stage --no-cpu-baseline > gpurun_out/bench_stage.json 2> gpurun_out/bench_stage.err; tail -c 2500 gpurun_out/bench_stage.json; tail -5 gpurun_out/bench_stage.err
timeout 600 python bench.py --stage --no-cpu-baseline --no-e2e --grad-precision bf16 > gpurun_out/bench_stage_bf16.json 2>&1; tail -c 300 gpurun_out/bench_stage_bf16.json
