# A/B under the power cap: TMA L2 cache hints of the fused passes (KD_L2_HINTS bits; 0 = default).
for rep in 1 2; do for h in 0 1 3 8; do
  KD_L2_HINTS=$h timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-variants > gpurun_out/l2h_$h.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/l2h_$h.json').read().strip().splitlines()[-1]); k=d['kernels']; print('hints=$h', round(d['value']), d['clocks']['sm_mhz'], d['clocks']['power_w_max'], {n: round(k[n]['ms_per_step'],2) for n in ('pass1','pass2','gemm_dh')})"
done; done
