export PYTHONUNBUFFERED=1
for r in a b c; do
KD_LIB_PATH=$PWD/paper_2603_01875_b200/libkdfused_r1.so timeout 300 python bench.py --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ab_r1$r.json 2> gpurun_out/ab_r1$r.err
timeout 300 python bench.py --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ab_cur$r.json 2> gpurun_out/ab_cur$r.err
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/ab_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    k=d.get("kernels",{})
    print(f, round(d["value"]), round(d["ms_per_step"],2), {n:round(v["ms_per_step"],2) for n,v in list(k.items())[:5]}, d["clocks"].get("sm_mhz"), d["clocks"].get("samples"), round(d["roofline"]["frac"],3))
P
