# Same-box A/B of the dh GEMM promotion period (KD_KB_PER_ACC) now that its slab tiles stay in L2, plus the parity
# ratios of the gradient tests that carry allowances at the shorter period
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/ab9
for r in a b c; do
for k in 64 32 16; do
  KD_KB_PER_ACC=$k timeout 300 python bench.py --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ab9/kb${k}_$r.json 2>/dev/null
done
done
python - <<'P'
import json,glob,collections
agg=collections.defaultdict(list)
for f in sorted(glob.glob("gpurun_out/ab9/kb*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); k=d.get("kernels",{})
    v=f.split("/")[-1].split("_")[0]; agg[v].append(d["value"])
    print(f, round(d["value"]), {n:round(x["ms_per_step"],2) for n,x in list(k.items())[:4]}, d["clocks"].get("sm_mhz"))
for v,x in sorted(agg.items()): print(v, round(sum(x)/len(x)))
P
for k in 64 16; do
  rm -f gpurun_out/ab9/parity_kb$k.jsonl
  KD_KB_PER_ACC=$k KD_PARITY_LOG=$PWD/gpurun_out/ab9/parity_kb$k.jsonl timeout 1200 python -m pytest tests/test_gpu_full.py tests/test_gpu_general.py -q --tb=line -k "reduced_n or sharp_temperature or config5_real" > gpurun_out/ab9/tests_kb$k.log 2>&1; echo "kb$k tests rc=$?"; tail -2 gpurun_out/ab9/tests_kb$k.log
  python - gpurun_out/ab9/parity_kb$k.jsonl <<'P'
import json,sys
for l in open(sys.argv[1]):
    r=json.loads(l)
    if r["strict_violations"] or r["max_err_over_strict_tol"]>0.8: print(r["test"].split("::")[-1], r["name"], round(r["max_err_over_strict_tol"],3), r["strict_violations"])
P
done
