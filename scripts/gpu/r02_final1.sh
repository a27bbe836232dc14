# Round-2 evidence: GPU test suite with the parity log, default bench (full line), other configs, launch list, ncu
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
rm -f gpurun_out/parity_final.jsonl
KD_PARITY_LOG=$PWD/gpurun_out/parity_final.jsonl timeout 1800 python -m pytest tests -m gpu -q --tb=short -rf > gpurun_out/gpu_tests_final.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/gpu_tests_final.log
timeout 900 python bench.py --graph > gpurun_out/bench_final_default.json 2> gpurun_out/bench_final_default.err; echo "bench rc=$?"
for c in c3_rkl c3_jsd c4 c5; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-variants > gpurun_out/bench_final_$c.json 2> gpurun_out/bench_final_$c.err; echo "$c rc=$?"; done
timeout 600 python bench.py --sim-vocab-shards 8 --no-cpu-baseline --no-variants --no-e2e > gpurun_out/bench_final_simv8.json 2> gpurun_out/bench_final_simv8.err; echo "simv8 rc=$?"
timeout 600 python bench.py --handoff --no-cpu-baseline --no-variants > gpurun_out/bench_final_handoff.json 2> gpurun_out/bench_final_handoff.err; echo "handoff rc=$?"
# launch list of the default bench command (per-launch times, cold-cache, serialised)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --no-variants --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu launches rc=$?"
# full sets of the three tensor kernels at one 2048-token chunk of c2
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"kd_pass_kernel|kd_gemm_kernel" -c 3 -o gpurun_out/r02_full python bench.py --tokens 2048 --steps 1 --warmup 1 --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i gpurun_out/r02_full.ncu-rep --page raw --csv > gpurun_out/r02_full_raw.csv 2>/dev/null; echo "export rc=$?"
