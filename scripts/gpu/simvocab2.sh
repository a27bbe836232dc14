timeout 900 python -m pytest tests/test_gpu_full.py -q --tb=short -k "vocab" > gpurun_out/vocab_tests.log 2>&1; tail -2 gpurun_out/vocab_tests.log
for spec in "c3_jsd 2" "c3_jsd 8"; do set -- $spec
  timeout 900 python bench.py --config $1 --sim-vocab-shards $2 --steps 5 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/bench_simv_$1_$2.json 2> gpurun_out/bench_simv_$1_$2.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_simv_$1_$2.json').read().strip().splitlines()[-1]); v=d['vocab_sharded']
print('$1 P=$2', 'token-sharded', round(d['value']), round(d['ms_per_step'],1), 'ms | vocab rank 0', round(v['ms_per_step'],1), 'ms, job excl comm', round(v['value']), 'eff', round(d['ms_per_step']/v['ms_per_step'],3), 'MHz', d['clocks']['sm_mhz'], {k: round(x,2) for k,x in v['kernels_ms_per_step'].items()})"
  tail -1 gpurun_out/bench_simv_$1_$2.err
done
