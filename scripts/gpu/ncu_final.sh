# ncu --set full of the three tensor kernels of the default path (one 2048-token chunk at c2), current code.
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"kd_pass_kernel|kd_gemm_kernel" -c 3 \
  -o gpurun_out/r01_full_final python bench.py --tokens 2048 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-variants > gpurun_out/ncu_final.log 2>&1; tail -2 gpurun_out/ncu_final.log
ls -la gpurun_out/r01_full_final.ncu-rep
