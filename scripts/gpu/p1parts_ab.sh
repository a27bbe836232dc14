# A/B under the power cap: pass-1 epilogue warps per TMEM lane quarter (3 = default, 2).
L=$PWD/paper_2603_01875_b200
KD_LIB_PATH=$L/libkdfused_p1e2.so timeout 900 python -m pytest tests/test_gpu_parity.py -q --tb=short -x > gpurun_out/p1e2_tests.log 2>&1; tail -1 gpurun_out/p1e2_tests.log
for rep in 1 2 3; do for v in base p1e2; do
  lib=$L/libkdfused.so; [ $v != base ] && lib=$L/libkdfused_$v.so
  KD_LIB_PATH=$lib timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/p1_$v.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/p1_$v.json').read().strip().splitlines()[-1]); k=d['kernels']; print('$v', round(d['value']), d['clocks']['sm_mhz'], {n: round(k[n]['ms_per_step'],2) for n in ('pass1','pass2','gemm_dh')}, 'staged', round(d['staged_variant']['value']))"
done; done
