# A/B under the power cap: nanosleep backoff in the mbarrier wait loops (KD_WAIT_BACKOFF_NS 0 = default).
L=$PWD/paper_2603_01875_b200
for rep in 1 2; do for v in base bo32 bo200; do
  lib=$L/libkdfused.so; [ $v != base ] && lib=$L/libkdfused_$v.so
  KD_LIB_PATH=$lib timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bo_$v.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bo_$v.json').read().strip().splitlines()[-1]); k=d['kernels']; print('$v', round(d['value']), d['clocks']['sm_mhz'], d['clocks']['power_w_max'], {n: round(k[n]['ms_per_step'],2) for n in ('pass1','pass2','gemm_dh')}, 'staged', round(d['staged_variant']['value']))"
done; done
