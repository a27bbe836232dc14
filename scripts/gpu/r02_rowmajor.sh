export PYTHONUNBUFFERED=1
L=$PWD/paper_2603_01875_b200
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stage.py tests/test_gpu_topk.py tests/test_gpu_lse.py tests/test_gpu_full.py -m gpu -q -x --tb=short > gpurun_out/rm_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/rm_tests.log
for r in a b c; do
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab13_rm$r.json 2>/dev/null
KD_LIB_PATH=$L/libkdfused_head.so timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab13_head$r.json 2>/dev/null
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/ab13_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    k=d.get("kernels",{})
    print(f, round(d["value"]), round(d["ms_per_step"],2), {n:round(v["ms_per_step"],2) for n,v in list(k.items())[:5]}, d["clocks"].get("sm_mhz"), "staged", round(d["staged_variant"]["value"]), {n:round(v["ms_per_step"],2) for n,v in list(d["staged_variant"]["kernels"].items())[:4]})
P
