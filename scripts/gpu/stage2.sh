# Staged variant: full parity file + ncu of the staged G kernel and the staged pass 1 (one 2048-token chunk).
timeout 1500 python -m pytest tests/test_gpu_stage.py -q --tb=short > gpurun_out/stage_tests.log 2>&1; tail -8 gpurun_out/stage_tests.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_stage_grad|kd_pass_kernel" -c 2 \
  -o gpurun_out/r01_stage_full python bench.py --stage --tokens 2048 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_stage.log 2>&1; tail -3 gpurun_out/ncu_stage.log
ls -la gpurun_out/
