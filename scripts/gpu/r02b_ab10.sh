# Same-box A/B: pass-2 G stores evict_first (KD_X_G_FIRST) vs the final build
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/ab10
KD_LIB_PATH=$PWD/paper_2603_01875_b200/libkdfused_gf.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --tb=short > gpurun_out/ab10/parity_gf.log 2>&1; echo "(gf) parity rc=$?"; tail -1 gpurun_out/ab10/parity_gf.log
for r in a b c d; do
for v in def gf; do
  if [ $v = def ]; then L=$PWD/paper_2603_01875_b200/libkdfused.so; else L=$PWD/paper_2603_01875_b200/libkdfused_$v.so; fi
  KD_LIB_PATH=$L timeout 300 python bench.py --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ab10/${v}_$r.json 2>/dev/null
done
done
for v in def gf; do
  if [ $v = def ]; then L=$PWD/paper_2603_01875_b200/libkdfused.so; else L=$PWD/paper_2603_01875_b200/libkdfused_$v.so; fi
  KD_LIB_PATH=$L timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"kd_pass_kernel|kd_gemm" --launch-skip 6 -c 6 --csv python bench.py --tokens 6144 --steps 1 --warmup 1 --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ab10/ncu_$v.csv 2>/dev/null; echo "ncu $v rc=$?"
done
python - <<'P'
import json,glob,collections
agg=collections.defaultdict(list)
for f in sorted(glob.glob("gpurun_out/ab10/*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); k=d.get("kernels",{})
    v=f.split("/")[-1].split("_")[0]; agg[v].append(d["value"])
    print(f, round(d["value"]), {n:round(x["ms_per_step"],2) for n,x in list(k.items())[:4]}, d["clocks"].get("sm_mhz"), d["clocks"].get("power_w_median"))
for v,x in sorted(agg.items()): print(v, round(sum(x)/len(x)))
P
