timeout 900 python -m pytest tests/test_gpu_stage.py tests/test_gpu_handoff.py -q --tb=short > gpurun_out/stage_edge.log 2>&1; tail -15 gpurun_out/stage_edge.log
