# Hand-off (NEXT-4) test + default bench line (with the staged-variant leg) + hand-off leg.
timeout 600 python -m pytest tests/test_gpu_handoff.py tests/test_gpu_stage.py -q --tb=short > gpurun_out/handoff_tests.log 2>&1; tail -4 gpurun_out/handoff_tests.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 1200 gpurun_out/bench_default.json; tail -3 gpurun_out/bench_default.err
timeout 900 python bench.py --handoff --no-variants --no-e2e --no-cpu-baseline > gpurun_out/bench_handoff.json 2> gpurun_out/bench_handoff.err; tail -c 1200 gpurun_out/bench_handoff.json; tail -3 gpurun_out/bench_handoff.err
