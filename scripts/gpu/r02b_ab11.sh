# Vocab-sharded exchange chunk vs the 3072-token library chunk: P = 8 simulated on one GPU (rank 0's compute)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/ab11
for r in a b; do
for x in def 6144 9216; do
  E=""; [ $x != def ] && E="KD_VOCAB_FIX_CHUNK=$x"
  env $E timeout 600 python bench.py --sim-vocab-shards 8 --no-cpu-baseline --no-variants --no-e2e > gpurun_out/ab11/simv8_${x}_$r.json 2>/dev/null
done; done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/ab11/*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); v=d["vocab_sharded"]
    print(f, round(d["value"]), round(v["value"]), round(v["ms_per_step"],2), round(v["strong_scaling_efficiency_excl_comm"],3), v.get("exchange_chunk_tokens"), d["clocks"].get("sm_mhz"))
P
