# Same-box A/B under the power cap: decoupled pass 2 (default) vs coupled pass 2 (no staging traffic) vs die-aware
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for r in a b c; do
for v in base coupled die; do
  case $v in base) E="";; coupled) E="KD_P2_COUPLED=1";; die) E="KD_DIE_SCHED=1";; esac
  env $E timeout 300 python bench.py --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ab1_${v}_$r.json 2>/dev/null
done
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/ab1_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    k=d.get("kernels",{})
    print(f, round(d["value"]), round(d["ms_per_step"],2), {n:round(v["ms_per_step"],2) for n,v in list(k.items())[:4]}, d["clocks"].get("sm_mhz"), d["clocks"].get("power_w_max"))
P
