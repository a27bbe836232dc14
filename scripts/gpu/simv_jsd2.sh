for C in 4096 8192; do
KD_VOCAB_FIX_CHUNK=$C timeout 900 python bench.py --config c3_jsd --sim-vocab-shards 2 --steps 3 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/bench_simv2_jsd_$C.json 2> gpurun_out/bench_simv2_jsd_$C.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_simv2_jsd_$C.json').read().strip().splitlines()[-1]); v=d['vocab_sharded']
print('chunk $C', round(d['ms_per_step'],1), round(v['ms_per_step'],1), 'eff', round(d['ms_per_step']/v['ms_per_step'],3), {k: round(x,2) for k,x in v['kernels_ms_per_step'].items()})"
tail -1 gpurun_out/bench_simv2_jsd_$C.err
done
