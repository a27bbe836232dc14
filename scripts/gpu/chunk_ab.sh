# A/B under the power cap: token chunk of the default path (KD_CHUNK_TOKENS; default 2048 at c2) and the coupled pass 2.
for rep in 1 2; do for v in "KD_CHUNK_TOKENS=2048" "KD_CHUNK_TOKENS=1024" "KD_CHUNK_TOKENS=4096" "KD_P2_COUPLED=1"; do
  env $v timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ck.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ck.json').read().strip().splitlines()[-1]); k=d['kernels']; print('$v', round(d['value']), d['clocks']['sm_mhz'], {n: round(k[n]['ms_per_step'],2) for n in ('pass1','pass2','gemm_dh')}, 'staged', round(d['staged_variant']['value']))"
done; done
