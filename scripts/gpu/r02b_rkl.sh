# RKL pass 1 decoupled with the teacher half staged: full GPU suite (parity log), then same-box A/B vs the coupled form
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/rkl
rm -f gpurun_out/rkl/parity.jsonl
KD_PARITY_LOG=$PWD/gpurun_out/rkl/parity.jsonl timeout 1800 python -m pytest tests -m gpu -q --tb=short -rf > gpurun_out/rkl/gpu_tests.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/rkl/gpu_tests.log
for r in a b c; do
for c in c3_rkl c5; do
for v in dec cpl; do
  E=""; [ $v = cpl ] && E="KD_RKL_P1_COUPLED=1"
  env $E timeout 300 python bench.py --config $c --no-variants --no-cpu-baseline --no-e2e > gpurun_out/rkl/${c}_${v}_$r.json 2>/dev/null
done; done; done
python - <<'P'
import json,glob,collections
agg=collections.defaultdict(list)
for f in sorted(glob.glob("gpurun_out/rkl/c*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); k=d.get("kernels",{})
    v=f.split("/")[-1].rsplit("_",1)[0]; agg[v].append(d["value"])
    print(f, round(d["value"]), {n:round(x["ms_per_step"],2) for n,x in list(k.items())[:4]}, d["clocks"].get("sm_mhz"))
for v,x in sorted(agg.items()): print(v, round(sum(x)/len(x)))
P
