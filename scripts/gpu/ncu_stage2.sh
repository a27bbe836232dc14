# ncu --set full of k_stage_grad v2 (one 2048-token chunk at c2), the staged path's HBM-bound kernel.
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_stage_grad" -c 1 \
  -o gpurun_out/r01_stage_v2 python bench.py --stage --tokens 2048 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_stage2.log 2>&1; tail -2 gpurun_out/ncu_stage2.log
ls -la gpurun_out/r01_stage_v2.ncu-rep
