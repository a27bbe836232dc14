# A/B: decoupled pass 2 staging the teacher half-tile in shared memory (3-stage ring) vs L2 (7-stage ring).
L=$PWD/paper_2603_01875_b200
KD_LIB_PATH=$L/libkdfused_p2smem.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stage.py -q --tb=short -x -k "not full_size" > gpurun_out/p2smem_tests.log 2>&1; tail -2 gpurun_out/p2smem_tests.log
for rep in 1 2; do for v in base p2smem; do
  lib=$L/libkdfused.so; [ $v = p2smem ] && lib=$L/libkdfused_p2smem.so
  KD_LIB_PATH=$lib timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-variants > gpurun_out/ab_$v.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]); k=d['kernels']; print('$v', round(d['value']), d['clocks']['sm_mhz'], {n: round(k[n]['ms_per_step'],2) for n in ('pass1','pass2','gemm_dh')}, round(d['roofline']['frac'],3))"
done; done
