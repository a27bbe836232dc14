export PYTHONUNBUFFERED=1
L=$PWD/paper_2603_01875_b200
for r in a b; do
timeout 300 python bench.py --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ab9_cur$r.json 2>/dev/null
KD_LIB_PATH=$L/libkdfused_tree.so timeout 300 python bench.py --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ab9_tree$r.json 2>/dev/null
KD_LIB_PATH=$L/libkdfused_resid.so timeout 300 python bench.py --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ab9_resid$r.json 2>/dev/null
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/ab9_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    k=d.get("kernels",{})
    print(f, round(d["value"]), round(d["ms_per_step"],2), {n:round(v["ms_per_step"],2) for n,v in list(k.items())[:5]}, d["clocks"].get("sm_mhz"), d["clocks"].get("power_w_max"))
P
