export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/chk
timeout 900 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_full.py -q --tb=short -rf -k "p2p or vocab" > gpurun_out/chk/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/chk/tests.log
timeout 600 python bench.py --sim-vocab-shards 8 --no-cpu-baseline --no-variants --no-e2e > gpurun_out/chk/simv8.jsonl 2>/dev/null; echo "simv8 rc=$?"
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/chk/default.jsonl 2>/dev/null; echo "default rc=$?"
python - <<'P'
import json
for f in ("gpurun_out/chk/simv8.jsonl","gpurun_out/chk/default.jsonl"):
    d=json.loads(open(f).read().strip().splitlines()[-1]); v=d["vocab_sharded"]
    print(f, round(d["value"]), round(v["value"]), round(v["ms_per_step"],2), v.get("strong_scaling_efficiency_excl_comm"), v.get("vs_fused_single_call"), v.get("exchange_chunk_tokens"), d.get("p2p_one_gpu",{}).get("value"), d.get("p2p_one_gpu",{}).get("exchange_chunk_tokens"))
P
