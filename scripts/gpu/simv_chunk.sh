# Narrow vocab shard (P=8 simulated): library token chunk A/B (KD_CHUNK_TOKENS), FKL and RKL.
for C in 2048 4096 8192; do for cfg in c2 c3_rkl; do
  KD_CHUNK_TOKENS=$C timeout 900 python bench.py --config $cfg --sim-vocab-shards 8 --steps 3 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/simc_$cfg_$C.json 2> gpurun_out/simc.err
  python -c "
import json; d=json.loads(open('gpurun_out/simc_$cfg_$C.json').read().strip().splitlines()[-1]); v=d['vocab_sharded']
print('$cfg chunk $C', round(d['ms_per_step'],1), round(v['ms_per_step'],1), 'eff', round(d['ms_per_step']/v['ms_per_step'],3), d['clocks']['sm_mhz'], {k: round(x,2) for k,x in v['kernels_ms_per_step'].items()})"
done; done
