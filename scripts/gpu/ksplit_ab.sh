# A/B under the power cap: split-K factor of the dh GEMM (chosen 8 at c2; fewer slabs = less reduce traffic).
for rep in 1 2; do for k in 0 4 6; do
  KD_DH_KSPLIT=$k timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ks.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ks.json').read().strip().splitlines()[-1]); k=d['kernels']; print('ksplit=$k', round(d['value']), d['clocks']['sm_mhz'], {n: round(k[n]['ms_per_step'],2) for n in ('pass1','pass2','gemm_dh','reduce_dh')}, 'staged', round(d['staged_variant']['value']))"
done; done
