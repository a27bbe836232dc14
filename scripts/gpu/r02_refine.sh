export PYTHONUNBUFFERED=1
timeout 600 python scripts/probe_parity_src.py c2 c4 > gpurun_out/rf_probe.log 2>&1; grep -v "teacher logits" gpurun_out/rf_probe.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stage.py tests/test_gpu_full.py -m gpu -q -x --tb=short > gpurun_out/rf_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/rf_tests.log
for r in a b; do for f in 0 1; do KD_REFINE=$f timeout 300 python bench.py --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ab12_rf$f$r.json 2>/dev/null; done; done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/ab12_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    k=d.get("kernels",{})
    print(f, round(d["value"]), round(d["ms_per_step"],2), {n:round(v["ms_per_step"],2) for n,v in list(k.items())[:7]}, d["clocks"].get("sm_mhz"))
P
