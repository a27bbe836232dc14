timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -m gpu -q -x --tb=short -k "gemm or c2 or dW or accumulate or tiny or determinism" > gpurun_out/gpuq.log 2>&1; tail -2 gpurun_out/gpuq.log; grep -E "Error|error" gpurun_out/gpuq.log | head -5
run() { cfg=$1; shift; env "$@" timeout 300 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $BARGS > gpurun_out/b_x.log 2>&1; python - "$cfg $*" <<'PY'
import json,sys; d=json.loads(open("gpurun_out/b_x.log").read().strip().splitlines()[-1]); k=d["kernels"]; print(sys.argv[1], round(d["value"]), d["clocks"]["sm_mhz"], {n:round(v["ms_per_step"],2) for n,v in k.items() if v["ms_per_step"]>0.5}, {n:round(v.get("tensor_pipe_tflops_executed",0)) for n,v in k.items() if "gemm" in n})
PY
}
run c2; BARGS=--dW run c2; run c4
