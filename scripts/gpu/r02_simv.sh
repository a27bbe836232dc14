export PYTHONUNBUFFERED=1
for c in c2 c3_rkl c3_jsd; do for P in 2 4 8; do
  timeout 600 python bench.py --config $c --sim-vocab-shards $P --steps 10 --no-cpu-baseline --no-variants --no-e2e > gpurun_out/simv_${c}_$P.json 2> gpurun_out/simv_${c}_$P.err
done; done
KD_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29544 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/n2_gloo_final.json 2> gpurun_out/n2_gloo_final.err; echo "n2 rc=$?"
KD_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29545 bench.py --gpus 2 --config c3_jsd --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/n2_gloo_jsd.json 2> gpurun_out/n2_gloo_jsd.err; echo "n2 jsd rc=$?"
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/simv_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    v=d["vocab_sharded"]
    print(f, "1gpu", round(d["value"]), round(d["ms_per_step"],2), "| rank0", round(v["ms_per_step"],2), "ms job", round(v["value"]), "eff", round(v["strong_scaling_efficiency_excl_comm"],3), {n:round(x,2) for n,x in list(v["kernels_ms_per_step"].items())[:5]})
for f in ("gpurun_out/n2_gloo_final.json","gpurun_out/n2_gloo_jsd.json"):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d["value"], d["scaling"], d["config"]["parallelism"], d.get("token_sharded",{}).get("value"))
    except Exception as e: print(f, "ERR", e)
P
