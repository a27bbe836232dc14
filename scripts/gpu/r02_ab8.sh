export PYTHONUNBUFFERED=1
L=$PWD/paper_2603_01875_b200
for r in a b; do
timeout 300 python bench.py --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ab8_cur$r.json 2>/dev/null
KD_LIB_PATH=$L/libkdfused_resid.so timeout 300 python bench.py --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ab8_resid$r.json 2>/dev/null
KD_LIB_PATH=$L/libkdfused_c1.so KD_KB_PER_ACC=64 timeout 300 python bench.py --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ab8_c1$r.json 2>/dev/null
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/ab8_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    k=d.get("kernels",{})
    print(f, round(d["value"]), round(d["ms_per_step"],2), {n:round(v["ms_per_step"],2) for n,v in list(k.items())[:5]}, d["clocks"].get("sm_mhz"), d["clocks"].get("power_w_max"))
P
rm -f gpurun_out/parity8.jsonl
KD_PARITY_LOG=$PWD/gpurun_out/parity8.jsonl timeout 1800 python -m pytest tests -m gpu -q --tb=short -rf > gpurun_out/gpu_tests8.log 2>&1
echo "pytest rc=$?"; tail -8 gpurun_out/gpu_tests8.log
