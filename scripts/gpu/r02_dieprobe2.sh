export PYTHONUNBUFFERED=1
KD_DIE_DEBUG=2 timeout 300 python bench.py --tokens 4096 --steps 3 --no-variants --no-cpu-baseline --no-e2e > gpurun_out/dp_bench.json 2> gpurun_out/dp_bench.err; grep "kd: die" gpurun_out/dp_bench.err
for r in a b; do
timeout 300 python bench.py --steps 10 --no-variants --no-cpu-baseline --no-e2e > gpurun_out/b4_die1$r.json 2> gpurun_out/b4_die1$r.err
KD_DIE_SCHED=0 timeout 300 python bench.py --steps 10 --no-variants --no-cpu-baseline --no-e2e > gpurun_out/b4_die0$r.json 2> gpurun_out/b4_die0$r.err
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/b4_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    k=d.get("kernels",{})
    print(f, round(d["value"]), round(d["ms_per_step"],2), {n:round(v["ms_per_step"],2) for n,v in list(k.items())[:5]}, d["clocks"].get("sm_mhz"), round(d["roofline"]["frac"],3))
P
for dsch in 1 0; do
KD_DIE_SCHED=$dsch timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:kd_pass_kernel -s 4 -c 4 --csv python bench.py --tokens 4096 --steps 1 --warmup 1 --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ncu2_die$dsch.csv 2> gpurun_out/ncu2_die$dsch.err
done
python - <<'P'
import csv
for d in (1,0):
    rows=list(csv.reader([l for l in open(f"gpurun_out/ncu2_die{d}.csv") if l.startswith('"')]))
    hdr=rows[0]
    for r in rows[1:]:
        rec=dict(zip(hdr,r))
        print("die",d, rec.get("Kernel Name","")[:28], rec.get("Metric Name"), rec.get("Metric Value"))
P
