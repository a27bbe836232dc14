# Round-end evidence (2): full GPU suite with the parity log, smoke(), default bench line, vocab-layout simulation.
KD_PARITY_LOG=gpurun_out/parity.jsonl timeout 2000 python -m pytest tests -m gpu -q --tb=short > gpurun_out/gpu_full.log 2>&1; tail -3 gpurun_out/gpu_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 300 gpurun_out/bench_default.json
for P in 2 8; do
  timeout 900 python bench.py --sim-vocab-shards $P --steps 5 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/bench_simv_c2_$P.json 2> gpurun_out/bench_simv_c2_$P.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_simv_c2_$P.json').read().strip().splitlines()[-1]); v=d['vocab_sharded']
print('c2 P=$P', 'token-sharded', round(d['value']), round(d['ms_per_step'],1), 'ms | vocab rank 0', round(v['ms_per_step'],1), 'ms, job excl comm', round(v['value']), 'eff', round(d['ms_per_step']/v['ms_per_step'],3), 'MHz', d['clocks']['sm_mhz'])"
done
