# Round 2 final evidence (+ RKL pass 1 staged): smoke, bench lines, launch list and ncu of the default build (the GPU suite of
# this build: scripts/gpu/r02b_rkl.sh)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/final5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final5/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/final5/smoke.log
timeout 900 python bench.py --graph > gpurun_out/final5/default.jsonl 2> gpurun_out/final5/default.err; echo "bench rc=$?"
for c in c3_rkl c3_jsd c4 c5; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-variants > gpurun_out/final5/$c.jsonl 2> gpurun_out/final5/$c.err; echo "$c rc=$?"; done
timeout 600 python bench.py --sim-vocab-shards 8 --no-cpu-baseline --no-variants --no-e2e > gpurun_out/final5/simv8.jsonl 2> gpurun_out/final5/simv8.err; echo "simv8 rc=$?"
timeout 600 python bench.py --sim-p2p 8 --steps 5 --no-cpu-baseline --no-variants --no-e2e > gpurun_out/final5/simp2p8.jsonl 2> gpurun_out/final5/simp2p8.err; echo "simp2p8 rc=$?"
timeout 600 python bench.py --handoff --no-cpu-baseline --no-variants > gpurun_out/final5/handoff.jsonl 2> gpurun_out/final5/handoff.err; echo "handoff rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final5/launches.csv python bench.py --steps 2 --warmup 3 --no-variants --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"kd_pass_kernel|kd_gemm_kernel|k_reduce_dh" --launch-skip 4 -c 4 -o gpurun_out/final5/full python bench.py --tokens 6144 --steps 1 --warmup 1 --no-variants --no-cpu-baseline --no-e2e > gpurun_out/final5/ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i gpurun_out/final5/full.ncu-rep --page raw --csv > gpurun_out/final5/full_raw.csv 2>/dev/null; echo "export rc=$?"
rm -f gpurun_out/final5/full.ncu-rep
