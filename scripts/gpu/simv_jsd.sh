# JSD vocab-shard path (P=8 simulated on one GPU): token chunk of the (K, J) exchange, A/B.
for C in 2048 8192; do
KD_VOCAB_FIX_CHUNK=$C timeout 900 python bench.py --config c3_jsd --sim-vocab-shards 8 --steps 3 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/bench_simv8_c3_jsd_$C.json 2> gpurun_out/bench_simv8_c3_jsd_$C.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_simv8_c3_jsd_$C.json').read().strip().splitlines()[-1]); v=d['vocab_sharded']
print('chunk $C', round(d['ms_per_step'],1), round(v['ms_per_step'],1), 'eff', round(d['ms_per_step']/v['ms_per_step'],3), 'host', round(v['host_enqueue_ms_per_step'],1), {k: round(x,2) for k,x in v['kernels_ms_per_step'].items()})"
tail -2 gpurun_out/bench_simv8_c3_jsd_$C.err
done
timeout 900 python bench.py --sim-vocab-shards 8 --steps 5 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/bench_simv8.json 2> gpurun_out/bench_simv8.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_simv8.json').read().strip().splitlines()[-1]); v=d['vocab_sharded']
print('fkl P=8', round(d['ms_per_step'],1), round(v['ms_per_step'],1), 'eff', round(d['ms_per_step']/v['ms_per_step'],3), 'host', round(v['host_enqueue_ms_per_step'],1))"
timeout 900 python bench.py --steps 5 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_quick.json').read().strip().splitlines()[-1]); print('default', round(d['value']), round(d['ms_per_step'],1), 'host', round(d['host_enqueue_ms_per_step'],2))"
