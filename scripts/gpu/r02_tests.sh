rm -f gpurun_out/parity.jsonl
KD_PARITY_LOG=$PWD/gpurun_out/parity.jsonl timeout 1800 python -m pytest tests -m gpu -q --tb=short -rf --durations=25 -s > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?"
tail -40 gpurun_out/gpu_tests.log
for k in 16 64; do KD_KB_PER_ACC=$k timeout 300 python bench.py --steps 10 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/bench_kb$k.json 2> gpurun_out/bench_kb$k.err; done
python - <<'P'
import json
for k in (16,64):
    d=json.loads(open(f"gpurun_out/bench_kb{k}.json").read().strip().splitlines()[-1])
    print(k, d["value"], d["ms_per_step"], {n:round(v["ms_per_step"],3) for n,v in d["kernels"].items()}, d["clocks"]["sm_mhz"])
P
