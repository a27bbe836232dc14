# pass-1 vs pass-2 in cycles + tensor-pipe activity (c2 shapes, one 4096-token chunk), then a full capture of pass 2
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__cycles_active.avg
timeout 600 ncu --metrics $M --clock-control none -k regex:kd_pass -c 4 --csv --log-file gpurun_out/ncu_pass_metrics.csv python bench.py --tokens 4096 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.DictReader(open("gpurun_out/ncu_pass_metrics.csv")))
for r in rows:
    print(r["ID"], r["Kernel Name"][:60], r["Metric Name"], r["Metric Value"])
PY
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kd_pass -s 1 -c 1 -o gpurun_out/pass2_full python bench.py --tokens 4096 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1; ls -la gpurun_out/*.ncu-rep
