run() { env "$@" timeout 300 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_x.log 2>&1; python - "$*" <<'PY'
import json,sys; d=json.loads(open("gpurun_out/b_x.log").read().strip().splitlines()[-1]); k=d["kernels"]; print(sys.argv[1], round(d["value"]), d["clocks"]["sm_mhz"], "p2/p1 %.3f" % (k["pass2"]["ms_per_step"]/k["pass1"]["ms_per_step"]), {n:round(v["ms_per_step"],2) for n,v in k.items() if v["ms_per_step"]>0.5})
PY
}
run KD_L2_HINTS=0
run KD_L2_HINTS=1
run KD_L2_HINTS=4
run KD_L2_HINTS=8
run KD_L2_HINTS=13
run KD_L2_HINTS=12
run KD_L2_HINTS=0 KD_CHUNK_TOKENS=2048
run KD_L2_HINTS=0 KD_CHUNK_TOKENS=8192
run KD_L2_HINTS=0
