export PYTHONUNBUFFERED=1
L=$PWD/paper_2603_01875_b200
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -m gpu -q -x --tb=short > gpurun_out/gtma_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gtma_tests.log
for r in a b; do
timeout 300 python bench.py --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ab6_gtma$r.json 2>/dev/null
KD_G_TMA=0 timeout 300 python bench.py --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ab6_scal$r.json 2>/dev/null
KD_LIB_PATH=$L/libkdfused_nogtma.so timeout 300 python bench.py --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ab6_nogtma$r.json 2>/dev/null
KD_LIB_PATH=$L/libkdfused_c1.so KD_KB_PER_ACC=64 timeout 300 python bench.py --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ab6_c1$r.json 2>/dev/null
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/ab6_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    k=d.get("kernels",{})
    print(f, round(d["value"]), round(d["ms_per_step"],2), {n:round(v["ms_per_step"],2) for n,v in list(k.items())[:5]}, d["clocks"].get("sm_mhz"), d["clocks"].get("power_w_max"))
P
