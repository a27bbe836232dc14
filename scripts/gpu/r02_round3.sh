set -x
export PYTHONUNBUFFERED=1
# 1. die map + the default bench (die-aware on) vs off, alternating
KD_DIE_DEBUG=1 timeout 300 python bench.py --steps 10 --no-variants --no-cpu-baseline --no-e2e > gpurun_out/b3_die1a.json 2> gpurun_out/b3_die1a.err
KD_DIE_SCHED=0 timeout 300 python bench.py --steps 10 --no-variants --no-cpu-baseline --no-e2e > gpurun_out/b3_die0a.json 2> gpurun_out/b3_die0a.err
timeout 300 python bench.py --steps 10 --no-variants --no-cpu-baseline --no-e2e > gpurun_out/b3_die1b.json 2> gpurun_out/b3_die1b.err
KD_DIE_SCHED=0 timeout 300 python bench.py --steps 10 --no-variants --no-cpu-baseline --no-e2e > gpurun_out/b3_die0b.json 2> gpurun_out/b3_die0b.err
grep "kd: die" gpurun_out/b3_die1a.err
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/b3_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    k=d.get("kernels",{})
    print(f, round(d["value"]), round(d["ms_per_step"],2), {n:round(v["ms_per_step"],2) for n,v in list(k.items())[:5]}, d["clocks"].get("sm_mhz"), d["clocks"].get("power_w_max"), round(d["roofline"]["frac"],3))
P
# 2. DRAM traffic of the fused passes, die-aware on / off (one 2048-token chunk, c2 shapes)
for dsch in 1 0; do
KD_DIE_SCHED=$dsch timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:kd_pass_kernel -c 6 --csv python bench.py --tokens 2048 --steps 1 --warmup 1 --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ncu_die$dsch.csv 2> gpurun_out/ncu_die$dsch.err
done
python - <<'P'
import csv
for d in (1,0):
    rows=list(csv.reader([l for l in open(f"gpurun_out/ncu_die{d}.csv") if l.startswith('"')]))
    hdr=rows[0]; 
    for r in rows[1:]:
        rec=dict(zip(hdr,r))
        print("die",d, rec.get("Kernel Name","")[:40], rec.get("Metric Name"), rec.get("Metric Value"))
P
# 3. the GPU test suite
KD_PARITY_LOG=$PWD/gpurun_out/parity3.jsonl timeout 1800 python -m pytest tests -m gpu -q --tb=short -rf -s > gpurun_out/gpu_tests3.log 2>&1
echo "pytest rc=$?"; grep -v "^\[parity\]" gpurun_out/gpu_tests3.log | tail -15; grep "^\[parity\]\|\.\[parity\]" gpurun_out/gpu_tests3.log | head -20
