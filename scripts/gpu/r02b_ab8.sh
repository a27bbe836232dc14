# Same-box A/B of the token chunk (KD_CHUNK_TOKENS) across configs, after the L2 hints
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
run() { cfg=$1; nc=$2; r=$3; shift 3; E=""; [ $nc != def ] && E="KD_CHUNK_TOKENS=$nc"
  env $E timeout 600 python bench.py --config $cfg --no-variants --no-cpu-baseline --no-e2e "$@" > gpurun_out/ab8_${cfg}_${nc}_$r.json 2>/dev/null; }
for r in a b; do
  for nc in def 2560 3072 3584; do run c2 $nc $r; done
  for nc in def 3072; do run c3_rkl $nc $r; run c5 $nc $r; done
  for nc in def 5120 6144; do run c4 $nc $r --steps 5; done
done
python - <<'P'
import json,glob,collections
agg=collections.defaultdict(list)
for f in sorted(glob.glob("gpurun_out/ab8_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    v=f.split("ab8_")[1].rsplit("_",1)[0]; agg[v].append((d["value"], d["clocks"].get("sm_mhz")))
    k=d.get("kernels",{})
    print(f, round(d["value"]), round(d["ms_per_step"],2), {n:round(x["ms_per_step"],2) for n,x in list(k.items())[:4]}, d["clocks"].get("sm_mhz"))
for v,x in sorted(agg.items()): print(v, round(sum(a for a,_ in x)/len(x)), [m for _,m in x])
P
