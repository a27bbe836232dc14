export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/final4
timeout 900 python bench.py > gpurun_out/final4/default.jsonl 2> gpurun_out/final4/default.err; echo "bench rc=$?"; tail -3 gpurun_out/final4/default.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/final4/default.jsonl").read().strip().splitlines()[-1])
print(round(d["value"]), d["ms_per_step"], d["clocks"], d["roofline"]["frac"])
p=d.get("p2p_one_gpu"); print({k:v for k,v in p.items() if k!="note"})
P
