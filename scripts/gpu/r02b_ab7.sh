# Same-box A/B after the L2 hints: staging split (smem chunks 2/3 vs 4), token chunk (3072/4096 vs 2048), die-aware
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for v in sch2 sch3; do KD_LIB_PATH=$PWD/paper_2603_01875_b200/libkdfused_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --tb=short > gpurun_out/ab7_parity_$v.log 2>&1; echo "($v) parity rc=$?"; tail -1 gpurun_out/ab7_parity_$v.log; done
for r in a b c; do
for v in def sch2 sch3 c3072 c4096 die; do
  L=$PWD/paper_2603_01875_b200/libkdfused.so; E=""
  case $v in sch2|sch3) L=$PWD/paper_2603_01875_b200/libkdfused_$v.so;; c3072) E="KD_CHUNK_TOKENS=3072";; c4096) E="KD_CHUNK_TOKENS=4096";; die) E="KD_DIE_SCHED=1";; esac
  env KD_LIB_PATH=$L $E timeout 300 python bench.py --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ab7_${v}_$r.json 2>/dev/null
done
done
python - <<'P'
import json,glob,collections
agg=collections.defaultdict(list)
for f in sorted(glob.glob("gpurun_out/ab7_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    k=d.get("kernels",{})
    v=f.split("ab7_")[1].rsplit("_",1)[0]; agg[v].append(d["value"])
    print(f, round(d["value"]), round(d["ms_per_step"],2), {n:round(x["ms_per_step"],2) for n,x in list(k.items())[:4]}, d["clocks"].get("sm_mhz"), d["clocks"].get("power_w_median"))
for v,x in agg.items(): print(v, round(sum(x)/len(x)))
P
