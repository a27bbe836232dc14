# Same-box A/B: the heads' TMA loads evict_last (pass 1 only / both passes) vs the default
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for v in wl1 wl; do KD_LIB_PATH=$PWD/paper_2603_01875_b200/libkdfused_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --tb=short > gpurun_out/ab6_parity_$v.log 2>&1; echo "($v) parity rc=$?"; tail -1 gpurun_out/ab6_parity_$v.log; done
for r in a b c; do
for v in def wl1 wl; do
  if [ $v = def ]; then L=$PWD/paper_2603_01875_b200/libkdfused.so; else L=$PWD/paper_2603_01875_b200/libkdfused_$v.so; fi
  KD_LIB_PATH=$L timeout 300 python bench.py --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ab6_${v}_$r.json 2>/dev/null
done
done
for v in def wl1 wl; do
  if [ $v = def ]; then L=$PWD/paper_2603_01875_b200/libkdfused.so; else L=$PWD/paper_2603_01875_b200/libkdfused_$v.so; fi
  KD_LIB_PATH=$L timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"kd_pass_kernel" --launch-skip 4 -c 4 --csv python bench.py --tokens 4096 --steps 1 --warmup 1 --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ab6_ncu_$v.csv 2>/dev/null; echo "ncu $v rc=$?"
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/ab6_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    k=d.get("kernels",{})
    print(f, round(d["value"]), round(d["ms_per_step"],2), {n:round(v["ms_per_step"],2) for n,v in list(k.items())[:4]}, d["clocks"].get("sm_mhz"), d["clocks"].get("power_w_median"))
P
