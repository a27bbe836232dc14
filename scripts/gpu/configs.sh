# Bench lines for the other BASELINE configs on one GPU (default path; staged leg included in each line).
timeout 900 python bench.py --config c4 --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -c 300 gpurun_out/bench_c4.json; tail -2 gpurun_out/bench_c4.err
timeout 900 python bench.py --config c5 --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -c 300 gpurun_out/bench_c5.json; tail -2 gpurun_out/bench_c5.err
timeout 900 python bench.py --dW --steps 5 --no-e2e > gpurun_out/bench_c2_dW.json 2> gpurun_out/bench_c2_dW.err; tail -c 300 gpurun_out/bench_c2_dW.json; tail -2 gpurun_out/bench_c2_dW.err
for f in c4 c5 c2_dW; do python -c "
import json; d=json.loads(open('gpurun_out/bench_$f.json').read().strip().splitlines()[-1]); print('$f', round(d['value']), d['clocks']['sm_mhz'], round(d['roofline']['frac'],3), round(d['useful_flop_frac'],3), 'staged', round(d['staged_variant']['value']), (d.get('cpu_baseline') or {}).get('single_thread'))"; done
