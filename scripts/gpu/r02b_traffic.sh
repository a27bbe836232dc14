# DRAM traffic per launch of the default path's kernels at the default 3072-token chunk: --metrics only, with
# ncu's cache flush between replays (default) and without (--cache-control none: the steady state of the step)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/traffic
for cc in all none; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control $cc -k regex:"kd_pass_kernel|kd_gemm|k_reduce_dh" --launch-skip 8 -c 8 --csv python bench.py --tokens 6144 --steps 1 --warmup 1 --no-variants --no-cpu-baseline --no-e2e > gpurun_out/traffic/ncu_$cc.csv 2>/dev/null; echo "ncu $cc rc=$?"
done
