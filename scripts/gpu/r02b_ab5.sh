# Same-box A/B: dh GEMM split-K slab tiles stored evict_last (KD_X_GEMM_SLAB_HINT) vs the default
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
KD_LIB_PATH=$PWD/paper_2603_01875_b200/libkdfused_gs.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -q -x --tb=short -k "c2 or tiny or self or edge or vocab" > gpurun_out/ab5_parity_gs.log 2>&1; echo "(gs) parity rc=$?"; tail -1 gpurun_out/ab5_parity_gs.log
for r in a b c; do
for v in base gs; do
  if [ $v = base ]; then L=$PWD/paper_2603_01875_b200/libkdfused.so; else L=$PWD/paper_2603_01875_b200/libkdfused_$v.so; fi
  KD_LIB_PATH=$L timeout 300 python bench.py --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ab5_${v}_$r.json 2>/dev/null
done
done
for v in base gs; do
  if [ $v = base ]; then L=$PWD/paper_2603_01875_b200/libkdfused.so; else L=$PWD/paper_2603_01875_b200/libkdfused_$v.so; fi
  KD_LIB_PATH=$L timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"kd_gemm_kernel|k_reduce_dh" --launch-skip 2 -c 2 --csv python bench.py --tokens 4096 --steps 1 --warmup 1 --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ab5_ncu_$v.csv 2>/dev/null; echo "ncu $v rc=$?"
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/ab5_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    k=d.get("kernels",{})
    print(f, round(d["value"]), round(d["ms_per_step"],2), {n:round(v["ms_per_step"],2) for n,v in list(k.items())[:4]}, d["clocks"].get("sm_mhz"), d["clocks"].get("power_w_median"))
P
for v in base gs; do echo "== $v"; grep -h '"kd_gemm\|"k_reduce' gpurun_out/ab5_ncu_$v.csv | python -c "
import sys,csv
for r in csv.reader(sys.stdin): print(r[4][:30], r[-3], r[-1])" ; done
