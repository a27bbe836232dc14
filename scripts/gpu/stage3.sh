# Staged variant: parity (R=4 default) + A/B of rows per thread in k_stage_grad + c3 kinds.
timeout 1500 python -m pytest tests/test_gpu_stage.py -q --tb=short > gpurun_out/stage_tests.log 2>&1; tail -4 gpurun_out/stage_tests.log
for R in 4 2 1; do
  lib=paper_2603_01875_b200/libkdfused.so; [ $R != 4 ] && lib=paper_2603_01875_b200/libkdfused_r$R.so
  KD_LIB_PATH=$PWD/$lib timeout 600 python bench.py --stage --no-cpu-baseline --no-e2e > gpurun_out/bench_stage_r$R.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_stage_r$R.json').read().strip().splitlines()[-1]); print('R=$R', round(d['value']), d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],2) for k,v in d['kernels'].items()}, round(d['kernels']['stage_grad']['achieved_GBps']))"
done
for c in c3_rkl c3_jsd; do
  timeout 600 python bench.py --config $c --stage --no-cpu-baseline --no-e2e > gpurun_out/bench_stage_$c.json 2>&1
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2>&1
  python -c "
import json
for f in ('gpurun_out/bench_stage_$c.json','gpurun_out/bench_$c.json'):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d['value']), d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],2) for k,v in d['kernels'].items()})"
done
