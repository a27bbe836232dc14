timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -m gpu -q -x --tb=short -k "not sharded" > gpurun_out/gpu11.log 2>&1; tail -3 gpurun_out/gpu11.log
for cfg in c2 c4 c3_jsd c3_rkl; do timeout 300 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_$cfg.log 2>&1; python - <<PY
import json; d=json.loads(open("gpurun_out/b_$cfg.log").read().strip().splitlines()[-1]); print("$cfg", round(d["value"]), d["clocks"]["sm_mhz"], {k:round(v["ms_per_step"],2) for k,v in d["kernels"].items()})
PY
done
KD_P2_COUPLED=1 timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_c4c.log 2>&1; python - <<PY
import json; d=json.loads(open("gpurun_out/b_c4c.log").read().strip().splitlines()[-1]); print("c4 coupled p2", round(d["value"]), d["clocks"]["sm_mhz"], {k:round(v["ms_per_step"],2) for k,v in d["kernels"].items()})
PY
