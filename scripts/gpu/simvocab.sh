# Vocab-sharded layout, compute of rank 0 of a P-way group simulated on one GPU (no exchange): per-GPU efficiency
# of the north star's primary layout vs the token-sharded (single-GPU) path, for P = 2, 4, 8.
for P in 2 4 8; do
  timeout 900 python bench.py --sim-vocab-shards $P --steps 5 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/bench_simv$P.json 2> gpurun_out/bench_simv$P.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_simv$P.json').read().strip().splitlines()[-1]); v=d['vocab_sharded']
print('P=$P', 'token-sharded 1-GPU', round(d['value']), 'ms', round(d['ms_per_step'],1), '| vocab rank-0 ms', round(v['ms_per_step'],1), 'job tok/s excl comm', round(v['value']), 'per-GPU eff', round(d['ms_per_step']/v['ms_per_step'],3), d['clocks']['sm_mhz'])"
  tail -2 gpurun_out/bench_simv$P.err
done
for c in c3_rkl c3_jsd; do
  timeout 900 python bench.py --config $c --sim-vocab-shards 8 --steps 3 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/bench_simv8_$c.json 2> gpurun_out/bench_simv8_$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_simv8_$c.json').read().strip().splitlines()[-1]); v=d['vocab_sharded']
print('$c P=8', round(d['value']), round(d['ms_per_step'],1), '| vocab', round(v['ms_per_step'],1), 'eff', round(d['ms_per_step']/v['ms_per_step'],3))"
  tail -2 gpurun_out/bench_simv8_$c.err
done
