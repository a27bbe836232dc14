# A/B of k_stage_grad shapes (rows x cols per thread, blocks per SM) inside the staged c2 step.
timeout 900 python -m pytest tests/test_gpu_stage.py -q --tb=short -x > gpurun_out/stage_tests.log 2>&1; tail -3 gpurun_out/stage_tests.log
for v in r4c4 r4c8 r2c8 r2c4; do
  lib=$PWD/paper_2603_01875_b200/libkdfused.so; [ $v != r4c4 ] && lib=$PWD/paper_2603_01875_b200/libkdfused_$v.so
  for bps in 4 8; do
    KD_STAGE_BPS=$bps KD_LIB_PATH=$lib timeout 600 python bench.py --stage --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/ab_$v_$bps.json 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/ab_$v_$bps.json').read().strip().splitlines()[-1]); k=d['kernels']; print('$v bps=$bps', round(d['value']), d['clocks']['sm_mhz'], round(k['stage_grad']['ms_per_step'],2), round(k['stage_grad']['achieved_GBps']), round(k['pass1']['ms_per_step'],2))"
  done
done
