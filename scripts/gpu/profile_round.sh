# Round-end evidence: full GPU suite, default bench line, ncu launch list of the bench command, and one
# `ncu --set full` capture of the three tensor kernels (one 2048-token chunk at c2 shapes).
set -x
timeout 1500 python -m pytest tests -m gpu -q --tb=short > gpurun_out/gpu_full.log 2>&1; tail -3 gpurun_out/gpu_full.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 600 gpurun_out/bench_default.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; wc -l gpurun_out/launches.csv
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"kd_pass_kernel|kd_gemm_kernel" -c 3 \
  -o gpurun_out/r01_full python bench.py --tokens 2048 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/
