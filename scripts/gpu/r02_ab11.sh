export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lse.py -m gpu -q -x --tb=short > gpurun_out/g11_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/g11_tests.log
for r in a b c; do
for g in 1 4; do KD_P1_GROUP=$g timeout 300 python bench.py --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ab11_g$g$r.json 2>/dev/null; done
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/ab11_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    k=d.get("kernels",{})
    print(f, round(d["value"]), round(d["ms_per_step"],2), {n:round(v["ms_per_step"],2) for n,v in list(k.items())[:5]}, d["clocks"].get("sm_mhz"), d["clocks"].get("power_w_max"))
P
for a in "c2 1.0" "c2 0.5" "c4 1.0"; do timeout 600 python scripts/probe_refine.py $a; done
